// k_rows.cu - A4/A5 row-list gather-attend for the fused path (GQA union rows)
// and A7 dense decode, with TMA-engine staging.
//
// One CTA owns a contiguous chunk of the row list of one (b, KV head g): either
// the union U_bg of the G q-heads' selected rows, each entry carrying the mask
// of q-heads that selected it (sd_sparse_decode_fused), or every row 0..N_b-1
// with all G heads (sd_dense_decode).  Each K/V row is fetched ONCE for the
// whole GQA group (union gather: the must-move bytes of SURVEY.md 8(d)).
//
// Staging: a producer warp resolves (page, slot) through the page table and
// issues one 1-D cp.async.bulk per 256-B row (K and V) into an NS-deep shared
// ring of 16-row stages; completion is counted in bytes on a per-stage
// mbarrier.  Four consumer warps (8 half-warps, one row each per step) read
// rows from shared memory, form the logits of the heads in the row's mask,
// and run the online softmax in the log2 domain (see k_attend.cu for the
// math).  Each CTA writes one unnormalised partial per q-head; the split merge
// is merge_parts_kernel.
#include "sd_common.cuh"
#include "sd_internal.h"
#include "sd_sbs.cuh"

namespace sd {
namespace {

constexpr int kStageRows = 16;
constexpr int kConsumerWarps = 4;
constexpr int kRowThreads = (kConsumerWarps + 1) * 32;

template <class KV>
struct RowCfg {
  static constexpr int kRowBytes = kD * KV::kBytes;
  static constexpr int kStages = KV::kBytes == 2 ? 8 : 4;
  static constexpr int kRingBytes = kStages * kStageRows * 2 * kRowBytes;
};

template <class KV>
__device__ __forceinline__ void lds_row8(const unsigned char* p, float* f) {
  if (KV::kBytes == 2) {
    unpack_bf16x8(*reinterpret_cast<const uint4*>(p), f);
  } else {
    const uint4 a = reinterpret_cast<const uint4*>(p)[0];
    const uint4 b = reinterpret_cast<const uint4*>(p)[1];
    f[0] = __uint_as_float(a.x); f[1] = __uint_as_float(a.y); f[2] = __uint_as_float(a.z); f[3] = __uint_as_float(a.w);
    f[4] = __uint_as_float(b.x); f[5] = __uint_as_float(b.y); f[6] = __uint_as_float(b.z); f[7] = __uint_as_float(b.w);
  }
}

template <class KV, int G, bool kDense>
__global__ void __launch_bounds__(kRowThreads) attend_rows_kernel(
    const void* __restrict__ q, const char* __restrict__ kp, const char* __restrict__ vp,
    const int* __restrict__ page_table, const int* __restrict__ seq_lens, int max_len, int max_pages, int Hkv,
    const uint32_t* __restrict__ fbm, int ldw, float scale_log2, float* __restrict__ part, int splits, int max_tok,
    int* __restrict__ err) {
  using Cfg = RowCfg<KV>;
  constexpr int RB = Cfg::kRowBytes;
  constexpr int NS = Cfg::kStages;
  extern __shared__ __align__(128) unsigned char smem[];
  unsigned char* ring = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Cfg::kRingBytes);
  uint64_t* empty = full + NS;
  int* s_pages = reinterpret_cast<int*>(empty + NS);                           // [max_tok / 16 + 1]
  constexpr int kW = kRangeTok / 32;
  uint32_t* bm = reinterpret_cast<uint32_t*>(s_pages + max_tok / 16 + 1);      // [G][kW]
  int* upre = reinterpret_cast<int*>(bm + (kDense ? 0 : G * kW));             // [kW + 1]
  __shared__ int warp_tot[kRowThreads / 32];

  const int bg = blockIdx.y, split = blockIdx.x;
  const int b = bg / Hkv, g = bg - b * Hkv;
  const int Hq = Hkv * G;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumerWarps);
    }
    fence_mbar_init();
  }
  const int hw = threadIdx.x >> 4, l16 = threadIdx.x & 15;
  float qf[G][8];
  if (warp < kConsumerWarps) {
#pragma unroll
    for (int j = 0; j < G; ++j) {
      load_q8<KV>(q, ((size_t)b * Hq + g * G + j) * kD + l16 * 8, qf[j]);
#pragma unroll
      for (int e = 0; e < 8; ++e) qf[j][e] *= scale_log2;
    }
  }
  const int Nr = seq_len_dev(seq_lens, b, max_len);  // out of range: an empty row
  if (kDense && Nr < 1 && split == 0 && g == 0 && threadIdx.x == 0) set_error(err, SD_DEVERR_SEQLEN);
  const int N = max(Nr, 0);
  int T0, T1;
  if (kDense) {
    int per = (N + splits - 1) / splits;
    per = (per + 15) & ~15;
    T0 = min(N, split * per);
    T1 = min(N, T0 + per);
  } else {
    T0 = min(N, split * kRangeTok);
    T1 = min(N, T0 + kRangeTok);
  }
  const int* pt = page_table + (size_t)b * max_pages;
  for (int i = threadIdx.x; i < ((T1 - T0 + 15) >> 4); i += kRowThreads) s_pages[i] = __ldg(pt + (T0 >> 4) + i);
  int nrows;
  const int nw = (T1 - T0 + 31) >> 5;
  if (kDense) {
    nrows = T1 - T0;
    __syncthreads();
  } else {
    pdl_wait();  // the selection bitmaps come from sbs_select_kernel
    nrows = T1 > T0 ? union_prologue<G, kRowThreads>(fbm, ldw, b * Hq + g * G, T0, T1, bm, upre, warp_tot) : 0;
  }
  const int r0 = 0, r1 = nrows;
  const int nst = (r1 - r0 + kStageRows - 1) / kStageRows;
  constexpr uint32_t kAll = (1u << G) - 1u;
  auto row_tl = [&](int i) -> int { return kDense ? i : union_row_token<G>(bm, upre, nw, i); };
  auto row_mask = [&](int i) -> uint32_t {
    if (kDense) return kAll;
    const int tl = row_tl(i);
    uint32_t mk = 0;
#pragma unroll
    for (int j = 0; j < G; ++j) mk |= ((bm[j * nw + (tl >> 5)] >> (tl & 31)) & 1u) << j;
    return mk;
  };
  auto row_index = [&](int i) -> uint32_t {
    const int t = T0 + row_tl(i);
    return (uint32_t)(s_pages[(t >> 4) - (T0 >> 4)] * kPS + (t & 15)) * (uint32_t)Hkv + (uint32_t)g;
  };

  float m[G], l[G], o[G][8];
#pragma unroll
  for (int j = 0; j < G; ++j) {
    m[j] = -INFINITY;
    l[j] = 0.f;
#pragma unroll
    for (int e = 0; e < 8; ++e) o[j][e] = 0.f;
  }

  if (warp == kConsumerWarps) {
    // ---------------- producer warp: one bulk copy per K or V row
    for (int s = 0; s < nst; ++s) {
      const int slot = s % NS;
      if (s >= NS) mbar_wait(&empty[slot], ((s / NS) - 1) & 1);
      const int base = s * kStageRows;
      const int cnt = min(kStageRows, (r1 - r0) - base);
      if (lane == 0) mbar_arrive_expect_tx(&full[slot], (uint32_t)(cnt * 2 * RB));
      __syncwarp();
      const int row = lane & 15, which = lane >> 4;
      if (row < cnt) {
        const size_t off = (size_t)row_index(base + row) * RB;
        bulk_g2s(ring + ((size_t)(slot * kStageRows + row) * 2 + which) * RB, (which ? vp : kp) + off, RB,
                 &full[slot]);
      }
    }
  } else {
    // ---------------- consumer warps: 8 half-warps, rows hw and hw + 8 of a stage
    for (int s = 0; s < nst; ++s) {
      const int slot = s % NS;
      const int base = s * kStageRows;
      const int cnt = min(kStageRows, (r1 - r0) - base);
      mbar_wait(&full[slot], (s / NS) & 1);
#pragma unroll
      for (int rr = 0; rr < 2; ++rr) {
        const int row = hw + rr * 8;
        const uint32_t mask = row < cnt ? row_mask(base + row) : 0u;
        const uint32_t need = __reduce_or_sync(0xffffffffu, mask);
        if (need == 0) continue;
        float kf[8], vf[8];
        const unsigned char* kr = ring + ((size_t)(slot * kStageRows + (row < cnt ? row : 0)) * 2) * RB +
                                  l16 * 8 * KV::kBytes;
        lds_row8<KV>(kr, kf);
        lds_row8<KV>(kr + RB, vf);
#pragma unroll
        for (int j = 0; j < G; ++j) {
          if (!((need >> j) & 1u)) continue;
          float sj = 0.f;
#pragma unroll
          for (int e = 0; e < 8; ++e) sj = fmaf(qf[j][e], kf[e], sj);
          sj = half_warp_sum(sj);
          if ((mask >> j) & 1u) {
            if (sj > m[j]) {  // lazy rescale: only when the running max grows
              const float corr = exp2f(m[j] - sj);
              l[j] *= corr;
#pragma unroll
              for (int e = 0; e < 8; ++e) o[j][e] *= corr;
              m[j] = sj;
            }
            const float p = exp2f(sj - m[j]);
            l[j] += p;
#pragma unroll
            for (int e = 0; e < 8; ++e) o[j][e] = fmaf(p, vf[e], o[j][e]);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);
    }
  }
  __syncthreads();  // every stage consumed: the ring is free for the combine
  float* st_o = reinterpret_cast<float*>(smem);                    // [G][8][128]
  float* st_m = st_o + G * 8 * kD;                                  // [G][8]
  float* st_l = st_m + G * 8;                                       // [G][8]
  if (warp < kConsumerWarps) {
#pragma unroll
    for (int j = 0; j < G; ++j) {
#pragma unroll
      for (int e = 0; e < 8; ++e) st_o[(j * 8 + hw) * kD + l16 * 8 + e] = o[j][e];
      if (l16 == 0) {
        st_m[j * 8 + hw] = m[j];
        st_l[j * 8 + hw] = l[j];
      }
    }
  }
  __syncthreads();
  if (threadIdx.x < kD) {
    const int d = threadIdx.x;
    for (int j = 0; j < G; ++j) {
      float M = -INFINITY;
#pragma unroll
      for (int i = 0; i < 8; ++i) M = fmaxf(M, st_m[j * 8 + i]);
      float L = 0.f, O = 0.f;
      if (M != -INFINITY) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float mi = st_m[j * 8 + i];
          if (mi != -INFINITY) {
            const float c = exp2f(mi - M);
            L = fmaf(st_l[j * 8 + i], c, L);
            O = fmaf(st_o[(j * 8 + i) * kD + d], c, O);
          }
        }
      }
      float* dst = part + (((size_t)b * Hq + g * G + j) * splits + split) * kPartStride;
      dst[2 + d] = O;
      if (d == 0) {
        dst[0] = M;
        dst[1] = L;
      }
    }
  }
  if (!kDense) pdl_launch_dependents();
}

template <class KV, int G, bool kDense>
cudaError_t launch_rows_t(const Geo& g, const sd_paged_kv& kv, const void* q, const uint32_t* fbm, int ldw,
                          float scale, float* part, int splits, int* err, cudaStream_t st) {
  using Cfg = RowCfg<KV>;
  const int max_tok = kDense ? (((g.max_seq_len + splits - 1) / splits + 15) & ~15) : kRangeTok;
  const size_t smem = Cfg::kRingBytes + 2 * Cfg::kStages * sizeof(uint64_t) + sizeof(int) * (max_tok / 16 + 1) +
                      (kDense ? 0 : sizeof(uint32_t) * ((G + 1) * (kRangeTok / 32) + 1)) + 16;
  static_assert((size_t)Cfg::kRingBytes >= (size_t)G * 8 * (kD + 2) * 4, "combine scratch must fit the ring");
  auto kern = attend_rows_kernel<KV, G, kDense>;
  cudaError_t e = ensure_dyn_smem(reinterpret_cast<const void*>(kern), smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(splits, g.B * g.Hkv);
  cfg.blockDim = dim3(kRowThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = kDense ? 0 : 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, q, reinterpret_cast<const char*>(kv.k_pages),
                            reinterpret_cast<const char*>(kv.v_pages), kv.page_table, kv.seq_lens, g.max_seq_len,
                            g.max_pages, g.Hkv, fbm, ldw, scale * kLog2e, part, splits, max_tok, err);
}

template <class KV, bool kDense>
cudaError_t launch_rows_g(const Geo& g, const sd_paged_kv& kv, const void* q, const uint32_t* fbm, int ldw,
                          float scale, float* part, int splits, int* err, cudaStream_t st) {
  switch (g.G) {
    case 1: return launch_rows_t<KV, 1, kDense>(g, kv, q, fbm, ldw, scale, part, splits, err, st);
    case 2: return launch_rows_t<KV, 2, kDense>(g, kv, q, fbm, ldw, scale, part, splits, err, st);
    case 4: return launch_rows_t<KV, 4, kDense>(g, kv, q, fbm, ldw, scale, part, splits, err, st);
    case 8: return launch_rows_t<KV, 8, kDense>(g, kv, q, fbm, ldw, scale, part, splits, err, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace

// fp32 KV only (the bf16 paths run on the tensor cores: k_attend_pk.cu, k_rows_mma.cu)
cudaError_t launch_attend_rows(const Geo& g, const sd_paged_kv& kv, const void* q, const uint32_t* fbm, int ldw,
                               float scale, float* part, int splits, cudaStream_t st) {
  if (g.kv_dtype != SD_F32) return cudaErrorInvalidValue;
  return launch_rows_g<KvF32, false>(g, kv, q, fbm, ldw, scale, part, splits, nullptr, st);
}

cudaError_t launch_dense_rows(const Geo& g, const sd_paged_kv& kv, const void* q, float scale, float* part,
                              int splits, int* err, cudaStream_t st) {
  if (g.kv_dtype != SD_F32) return cudaErrorInvalidValue;
  return launch_rows_g<KvF32, true>(g, kv, q, nullptr, 0, scale, part, splits, err, st);
}

}  // namespace sd
