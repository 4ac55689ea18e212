// k_attend.cu - A4/A5 gather-attend over per-head index lists, A7 dense decode,
// and the split-k / cross-shard LSE merges.
//
// Math ("weighted attention given sparse index and associated weights";
// S:130-138; LSE S:124): s_i = scale <q, K_i>; the kernels work in the log2
// domain, x_i = s_i log2(e) + log2(w_i), and keep per split the running
//   m = max_i x_i,  l = sum_i 2^(x_i - m),  o = sum_i 2^(x_i - m) V_i
// (online softmax).  Splits are merged in split order (deterministic):
//   M = max m_s,  L = sum l_s 2^(m_s - M),  out = sum o_s 2^(m_s - M) / L,
//   lse = ln2 (M + log2 L) = log sum_i w_i e^{s_i}.
//
// Work mapping: a half-warp (16 lanes x 8 elements) owns one 128-wide K/V row;
// each lane keeps 8 output dims.  Rows are fetched with 16-B non-allocating
// vector loads straight from their page (page_table indirection);
// every loop iteration issues the loads of U rows per half-warp before any
// arithmetic so that ~U*512 B per half-warp are in flight.
#include <math.h>

#include "sd_common.cuh"
#include "sd_internal.h"
#include "sd_merge.cuh"

static_assert(sd::kMergeStride == sd::kPartStride, "merge helper and partial layout agree");

namespace sd {

namespace {

constexpr int kAttThreads = 128;           // 4 warps = 8 half-warps
constexpr int kHalfWarps = kAttThreads / 16;
constexpr int kUnroll = 2;

// Combine the 8 half-warp states of a CTA (smem) into one partial and store it.
__device__ __forceinline__ void cta_combine_store(float (*st_o)[kD], float* st_m, float* st_l,
                                                  float* dst) {
  const int d = threadIdx.x;  // 128 threads == 128 dims
  float M = -INFINITY;
#pragma unroll
  for (int i = 0; i < kHalfWarps; ++i) M = fmaxf(M, st_m[i]);
  float L = 0.f, O = 0.f;
  if (M != -INFINITY) {
#pragma unroll
    for (int i = 0; i < kHalfWarps; ++i) {
      if (st_m[i] != -INFINITY) {
        float c = exp2f(st_m[i] - M);
        L = fmaf(st_l[i], c, L);
        O = fmaf(st_o[i][d], c, O);
      }
    }
  }
  dst[2 + d] = O;
  if (d == 0) { dst[0] = M; dst[1] = L; }
}

// ---------------------------------------------------------------------------
// Gather-attend over per-(b, h) index lists (no GQA dedup; paper semantics).
// grid = (splits, B*Hq); block = 128.
// ---------------------------------------------------------------------------
template <class KV>
__global__ void __launch_bounds__(kAttThreads) attend_list_kernel(
    const void* __restrict__ q, const void* __restrict__ kp, const void* __restrict__ vp,
    const int* __restrict__ page_table, const int* __restrict__ seq_lens, int max_len, int max_pages,
    int Hq, int Hkv, const int* __restrict__ idx, const int* __restrict__ counts, int k_max,
    const float* __restrict__ weights, float scale_log2, float* __restrict__ part, int splits,
    int allow_empty, int* __restrict__ err) {
  __shared__ float st_o[kHalfWarps][kD];
  __shared__ float st_m[kHalfWarps], st_l[kHalfWarps];

  const int row = blockIdx.y, split = blockIdx.x;
  const int b = row / Hq, h = row - b * Hq, g = h / (Hq / Hkv);
  const int N = seq_len_dev(seq_lens, b, max_len);  // -1 (out of range): every count is rejected
  pdl_wait();  // idx / counts / weights may come from the preceding kernel (coherent loads below)
  int cnt = __ldcg(counts + row);
  if ((cnt < 1 && !allow_empty) || cnt > k_max || cnt > N) {
    if (split == 0 && threadIdx.x == 0) set_error(err, cnt < 1 ? SD_DEVERR_EMPTY : SD_DEVERR_SEQLEN);
    cnt = max(0, min(cnt, min(k_max, max(N, 0))));
  }
  const int per = (cnt + splits - 1) / splits;
  const int c0 = min(cnt, split * per), c1 = min(cnt, c0 + per);

  const int lane = threadIdx.x & 31, l16 = lane & 15;
  const int hw = threadIdx.x >> 4;
  float qf[8];
  load_q8<KV>(q, (size_t)row * kD + l16 * 8, qf);
#pragma unroll
  for (int j = 0; j < 8; ++j) qf[j] *= scale_log2;

  const int* ip = idx + (size_t)row * k_max;
  const float* wp = weights ? weights + (size_t)row * k_max : nullptr;
  const int* pt = page_table + (size_t)b * max_pages;

  float m = -INFINITY, l = 0.f, o[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) o[j] = 0.f;

  for (int it = c0; it < c1; it += kHalfWarps * kUnroll) {
    typename KV::Raw kr[kUnroll], vr[kUnroll];
    float xb[kUnroll];
    bool ok[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int e = it + u * kHalfWarps + hw;
      int t = 0;
      ok[u] = false;
      xb[u] = 0.f;
      if (e < c1) {
        t = __ldcg(ip + e);
        ok[u] = (t >= 0) && (t < N);
        if (ok[u] && e > 0 && __ldcg(ip + e - 1) >= t) {
          ok[u] = false;
          if (l16 == 0) set_error(err, SD_DEVERR_INDEX_ORDER);
        } else if (!ok[u] && l16 == 0) {
          set_error(err, SD_DEVERR_INDEX_RANGE);
        }
        if (ok[u] && wp) {
          const float w = __ldcg(wp + e);
          if (!(w > 0.f) || !isfinite(w)) {
            ok[u] = false;
            if (l16 == 0) set_error(err, SD_DEVERR_WEIGHT);
          } else {
            xb[u] = log2f(w);
          }
        }
        if (!ok[u]) t = 0;
      }
      const size_t re = kv_row_elem(__ldg(pt + (t >> 4)), t & 15, g, Hkv) + l16 * 8;
      kr[u] = KV::load(kp, re);
      vr[u] = KV::load(vp, re);
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      float kf[8];
      KV::unpack(kr[u], kf);
      float s = 0.f;
#pragma unroll
      for (int j = 0; j < 8; ++j) s = fmaf(qf[j], kf[j], s);
      s = half_warp_sum(s);
      if (ok[u]) {
        const float x = s + xb[u];
        const float mn = fmaxf(m, x);
        const float corr = exp2f(m - mn);
        const float p = exp2f(x - mn);
        float vf[8];
        KV::unpack(vr[u], vf);
        l = fmaf(l, corr, p);
#pragma unroll
        for (int j = 0; j < 8; ++j) o[j] = fmaf(o[j], corr, p * vf[j]);
        m = mn;
      }
    }
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) st_o[hw][l16 * 8 + j] = o[j];
  if (l16 == 0) { st_m[hw] = m; st_l[hw] = l; }
  __syncthreads();
  cta_combine_store(st_o, st_m, st_l, part + ((size_t)row * splits + split) * kPartStride);
}

// ---------------------------------------------------------------------------
// Split merge: grid = rows, block = 128 (one thread per output dim).
// Up to kMergeRegSplits splits (N <= 128K at 8192 tokens per split) take a
// register path with a single round of loads; more splits use shared memory.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(128) merge_parts_kernel(const float* __restrict__ part, int splits,
                                                          void* __restrict__ out, int out_dtype,
                                                          float* __restrict__ lse) {
  // splits <= blockDim.x * 4 (host-checked); all loads of a phase are independent
  __shared__ float s_c[4 * 128];
  __shared__ float s_red[2][4];
  const int row = blockIdx.x, d = threadIdx.x, lane = d & 31, warp = d >> 5;
  pdl_wait();  // no-op unless launched as a programmatic dependent
  const float* p = part + (size_t)row * splits * kPartStride;
  if (splits <= kMergeRegSplits) {
    merge_row_regs(part, splits, row, d, out, out_dtype, lse);
    return;
  }
  float mv[4], lv[4], M = -INFINITY;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int s = d + 128 * k;
    mv[k] = s < splits ? __ldcg(p + s * kPartStride) : -INFINITY;
    lv[k] = s < splits ? __ldcg(p + s * kPartStride + 1) : 0.f;
    M = fmaxf(M, mv[k]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
  if (lane == 0) s_red[0][warp] = M;
  __syncthreads();
  M = fmaxf(fmaxf(s_red[0][0], s_red[0][1]), fmaxf(s_red[0][2], s_red[0][3]));
  float L = 0.f;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int s = d + 128 * k;
    const float c = (M == -INFINITY || mv[k] == -INFINITY) ? 0.f : exp2f(mv[k] - M);
    if (s < splits) s_c[s] = c;
    L = fmaf(lv[k], c, L);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) L += __shfl_xor_sync(0xffffffffu, L, o);
  if (lane == 0) s_red[1][warp] = L;
  __syncthreads();
  L = (s_red[1][0] + s_red[1][1]) + (s_red[1][2] + s_red[1][3]);
  float O = 0.f;
#pragma unroll 8
  for (int s = 0; s < splits; ++s) O = fmaf(__ldcg(p + s * kPartStride + 2 + d), s_c[s], O);
  store_out(out, out_dtype, (size_t)row * kD + d, L > 0.f ? O / L : 0.f);
  if (lse && d == 0) lse[row] = L > 0.f ? (M + log2f(L)) * kLn2 : -INFINITY;
}

// Normalised parts (o_p, lse_p natural log) -> out, lse.  grid = rows.
__global__ void __launch_bounds__(128) lse_merge_kernel(int parts, int rows,
                                                        const float* __restrict__ po,
                                                        const float* __restrict__ pl,
                                                        void* __restrict__ out, int out_dtype,
                                                        float* __restrict__ lse) {
  const int row = blockIdx.x, d = threadIdx.x;
  float M = -INFINITY;
  for (int p = 0; p < parts; ++p) M = fmaxf(M, pl[(size_t)p * rows + row]);
  float L = 0.f, O = 0.f;
  if (M != -INFINITY) {
    for (int p = 0; p < parts; ++p) {
      const float lp = pl[(size_t)p * rows + row];
      if (lp != -INFINITY) {
        const float c = expf(lp - M);
        L += c;
        O = fmaf(po[((size_t)p * rows + row) * kD + d], c, O);
      }
    }
  }
  store_out(out, out_dtype, (size_t)row * kD + d, L > 0.f ? O / L : 0.f);
  if (lse && d == 0) lse[row] = L > 0.f ? M + logf(L) : -INFINITY;
}

}  // namespace

int choose_splits(int rows, int work_per_row, int min_per_split) {
  const int target = 148 * 8;  // CTAs: ~8 resident 128-thread CTAs per SM
  int s = (target + rows - 1) / max(rows, 1);
  int cap = (work_per_row + min_per_split - 1) / min_per_split;
  s = s < cap ? s : cap;
  if (s > kMaxSplits) s = kMaxSplits;
  if (s < 1) s = 1;
  return s;
}

cudaError_t launch_attend_list(const Geo& g, const sd_paged_kv& kv, const void* q,
                               const int* idx, const int* counts, int k_max,
                               const float* weights, float scale, float* part, int splits,
                               int allow_empty, int* err, cudaStream_t st) {
  const float sl2 = scale * kLog2e;
  // programmatic dependent launch: the launch overlaps the preceding kernel's tail
  // (the kernel waits for it before reading idx / counts / weights)
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(splits, g.B * g.Hq);
  cfg.blockDim = dim3(kAttThreads);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (g.kv_dtype == SD_BF16)
    return cudaLaunchKernelEx(&cfg, attend_list_kernel<KvBF16>, q, kv.k_pages, kv.v_pages, kv.page_table, kv.seq_lens,
                              g.max_seq_len, g.max_pages, g.Hq, g.Hkv, idx, counts, k_max, weights, sl2, part, splits,
                              allow_empty, err);
  return cudaLaunchKernelEx(&cfg, attend_list_kernel<KvF32>, q, kv.k_pages, kv.v_pages, kv.page_table, kv.seq_lens,
                            g.max_seq_len, g.max_pages, g.Hq, g.Hkv, idx, counts, k_max, weights, sl2, part, splits,
                            allow_empty, err);
}

cudaError_t launch_merge_parts(const float* part, int rows, int splits, void* out,
                               int out_dtype, float* lse, cudaStream_t st) {
  return launch_merge_parts_pdl(part, rows, splits, out, out_dtype, lse, st);
}

cudaError_t launch_merge_parts_pdl(const float* part, int rows, int splits, void* out, int out_dtype, float* lse,
                                   cudaStream_t st) {
  if (splits > 4 * 128) return cudaErrorInvalidValue;  // merge_parts_kernel bound
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(rows);
  cfg.blockDim = dim3(128);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, merge_parts_kernel, part, splits, out, out_dtype, lse);
}

cudaError_t launch_lse_merge(int parts, int rows, const float* part_o, const float* part_lse,
                             int out_dtype, void* out, float* lse, cudaStream_t st) {
  lse_merge_kernel<<<rows, 128, 0, st>>>(parts, rows, part_o, part_lse, out, out_dtype, lse);
  return cudaGetLastError();
}

}  // namespace sd
