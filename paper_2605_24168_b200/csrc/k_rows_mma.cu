// k_rows_mma.cu - A7 dense decode (the in-repo baseline) on
// the bf16 tensor cores.
//
// The G q-heads of one KV head share every gathered K/V row, so a 16-row tile
// is a real dense contraction (BASELINE north_star: "tensor cores ... where the
// GQA query group makes the selected-row QK^T/PV a real dense tile"):
//   S[16 x 16] = Q[16 (G heads + zero pad) x 128] . K_tile^T[128 x 16]
//   O[16 x 128] += P[16 x 16] . V_tile[16 x 128]
// with mma.sync m16n8k16 (bf16 in, fp32 accumulate).  K and V are exact bf16;
// P is split P = P_hi + P_lo into two bf16 terms (two PV mma's) so the output
// keeps ~fp32 accuracy.  Rows a head did not select are masked to -inf before
// the softmax (per-head selection bitmap of the CTA's token range).
//
// Each CTA owns one contiguous token range of one (b, g).
// Memory path: the range's page ids are cached in shared memory; rows are
// streamed into a 3-stage shared ring with 16-B cp.async (LDGSTS; rows past
// the end are zero-filled), XOR-swizzled per 16-B chunk so ldmatrix is
// bank-conflict-free.  Each of the 4 warps owns 16 rows of every 64-row stage
// and keeps its own online-softmax state; the 4 states are merged at the end
// into one unnormalised split-k partial per q-head, and the last CTA of each
// (b, g) merges the splits.
#include "sd_common.cuh"
#include "sd_internal.h"

namespace sd {
namespace {

constexpr int kMmaWarps = 4;
constexpr int kMmaThreads = kMmaWarps * 32;
constexpr int kTileRows = 16;
constexpr int kStageRowsM = kMmaWarps * kTileRows;   // 64 rows per stage
constexpr int kRowB = 256;                           // one bf16 K or V row
constexpr int kStageBytesM = kStageRowsM * 2 * kRowB;  // 32 KB (K block then V block)

__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool valid) {
  const uint32_t d = smem_u32(dst);
  const int n = valid ? 16 : 0;  // 0 => zero-fill
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
// D = A(16x16, row) * B(16x8, col) + D ; A rows 8..15 are zero (padding heads)
__device__ __forceinline__ void mma_bf16(float* d, uint32_t a0, uint32_t a2, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(0u), "r"(a2), "r"(0u), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
__device__ __forceinline__ float bf16_round(float x) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r << 16);
}

// swizzled byte offset of 16-B chunk c of row r inside a [rows][256 B] block
__device__ __forceinline__ uint32_t swz(int r, int c) { return (uint32_t)(r * kRowB + ((c ^ (r & 7)) << 4)); }

constexpr int kStagesM = 3;  // ring depth (2 stages in flight)

template <int G>
__global__ void __launch_bounds__(kMmaThreads) attend_rows_mma_kernel(
    const uint16_t* __restrict__ q, const char* __restrict__ kp, const char* __restrict__ vp,
    const int* __restrict__ page_table, const int* __restrict__ seq_lens, int max_len, int max_pages, int Hkv,
    float scale_log2, float* __restrict__ part, int splits, int max_tok, void* __restrict__ out, int out_dtype,
    float* __restrict__ lse_out, int* __restrict__ counters, int* __restrict__ err) {
  constexpr uint32_t kAll = (1u << G) - 1u;
  extern __shared__ __align__(128) unsigned char smem[];
  unsigned char* ring = smem;                                                     // [stages][K | V]
  int* s_pages = reinterpret_cast<int*>(ring + kStagesM * kStageBytesM);          // [max_tok / 16 + 1]

  const int bg = blockIdx.y, split = blockIdx.x;
  const int b = bg / Hkv, g = bg - b * Hkv;
  const int Hq = Hkv * G;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int qr = lane >> 2, qc2 = (lane & 3) * 2;  // fragment row (head) / column pair

  // Q as the A operand: 8 k-steps of 16 dims; rows >= G are zero
  uint32_t qa0[8], qa2[8];
#pragma unroll
  for (int kk = 0; kk < 8; ++kk) {
    qa0[kk] = 0u;
    qa2[kk] = 0u;
    if (qr < G) {
      const uint16_t* qrow = q + ((size_t)b * Hq + g * G + qr) * kD + kk * 16 + qc2;
      qa0[kk] = *reinterpret_cast<const uint32_t*>(qrow);
      qa2[kk] = *reinterpret_cast<const uint32_t*>(qrow + 8);
    }
  }
  const int Nr = seq_len_dev(seq_lens, b, max_len);
  if (Nr < 1 && split == 0 && tid == 0 && g == 0) set_error(err, SD_DEVERR_SEQLEN);  // row reads as empty
  const int N = max(Nr, 0);
  int per = (N + splits - 1) / splits;
  per = (per + 15) & ~15;
  const int T0 = min(N, split * per), T1 = min(N, T0 + per);  // token range of this CTA
  const int* pt = page_table + (size_t)b * max_pages;
  for (int i = tid; i < ((T1 - T0 + 15) >> 4); i += kMmaThreads) s_pages[i] = __ldg(pt + (T0 >> 4) + i);
  const int total = T1 - T0;
  __syncthreads();

  // coalesced cp.async issue: thread tid copies 16-B chunk tid % 16 of rows
  // tid / 16 + 8 i (i < 8) of the K and V blocks; the swizzled destination
  // chunk is the same for all of them ((tid / 16 + 8 i) & 7 == (tid / 16) & 7)
  const int ic = tid & 15, ir0 = tid >> 4;
  const uint32_t dsw = (uint32_t)(ir0 * kRowB + ((ic ^ (ir0 & 7)) << 4));
  const char* kpc = kp + ic * 16;
  const char* vpc = vp + ic * 16;
  const int p0 = T0 >> 4;

  float o[16][4];
#pragma unroll
  for (int i = 0; i < 16; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m = -INFINITY, lsum = 0.f;

  {
    const int nrows = total;
    const int nst = (nrows + kStageRowsM - 1) / kStageRowsM;
    auto issue = [&](int s) {
      if (s < nst) {
        unsigned char* st = ring + (size_t)(s % kStagesM) * kStageBytesM + dsw;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int r = s * kStageRowsM + ir0 + 8 * i;
          const bool valid = r < nrows;
          size_t off = 0;
          if (valid) {
            const int t = T0 + r;
            const uint32_t ri = (uint32_t)(s_pages[(t >> 4) - p0] * kPS + (t & 15)) * (uint32_t)Hkv + g;
            off = (size_t)ri * kRowB;
          }
          cp_async16(st + i * 8 * kRowB, kpc + off, valid);
          cp_async16(st + kStageRowsM * kRowB + i * 8 * kRowB, vpc + off, valid);
        }
      }
      cp_async_commit();
    };
#pragma unroll
    for (int s = 0; s < kStagesM - 1; ++s) issue(s);
    for (int s = 0; s < nst; ++s) {
      issue(s + kStagesM - 1);
      cp_async_wait<kStagesM - 1>();
      __syncthreads();
      const unsigned char* st = ring + (size_t)(s % kStagesM) * kStageBytesM;
      const int trow = warp * kTileRows;                 // this warp's tile inside the stage
      const int rbase = s * kStageRowsM + trow;          // batch-relative row of the tile
      if (rbase < nrows) {
        const uint32_t kb = smem_u32(st) + trow * kRowB;
        const uint32_t vb = smem_u32(st + kStageRowsM * kRowB) + trow * kRowB;
        // ---- S = Q K^T for the 16 rows (two n-tiles of 8 rows)
        float sc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
        const int lr = lane & 7, lm = lane >> 3;  // ldmatrix: row within matrix, matrix id
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const int r = (lm >> 1) * 8 + lr, c = 2 * kk + (lm & 1);
          uint32_t b0, b1, b2, b3;
          ldsm_x4(kb + swz(r, c), b0, b1, b2, b3);
          mma_bf16(sc[0], qa0[kk], qa2[kk], b0, b1);
          mma_bf16(sc[1], qa0[kk], qa2[kk], b2, b3);
        }
        // ---- masked online softmax for head qr (lanes qr >= G are padding)
        float x[4];
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int rr = rbase + nt * 8 + qc2 + e;
            const uint32_t mk = rr < nrows ? kAll : 0u;
            const bool ok = qr < G && ((mk >> qr) & 1u);
            x[nt * 2 + e] = ok ? sc[nt][e] * scale_log2 : -INFINITY;
          }
        }
        float tmax = fmaxf(fmaxf(x[0], x[1]), fmaxf(x[2], x[3]));
        tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 1));
        tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 2));
        const bool grow = tmax > m;
        if (__any_sync(0xffffffffu, grow)) {
          const float mn = grow ? tmax : m;
          const float corr = (m == -INFINITY) ? 0.f : exp2f(m - mn);
          lsum *= corr;
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            o[i][0] *= corr;
            o[i][1] *= corr;
          }
          m = mn;
        }
        float p[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) p[i] = (x[i] == -INFINITY) ? 0.f : exp2f(x[i] - m);
        lsum += (p[0] + p[1]) + (p[2] + p[3]);
        // P = P_hi + P_lo (bf16 each) -> A fragments (rows 8..15 zero)
        const uint32_t ph0 = pack_bf16(p[0], p[1]), ph2 = pack_bf16(p[2], p[3]);
        const uint32_t pl0 = pack_bf16(p[0] - bf16_round(p[0]), p[1] - bf16_round(p[1]));
        const uint32_t pl2 = pack_bf16(p[2] - bf16_round(p[2]), p[3] - bf16_round(p[3]));
        // ---- O += P V over 16 dim-tiles of 8
#pragma unroll
        for (int nd = 0; nd < 16; nd += 2) {
          const int r = (lm & 1) * 8 + lr, c = nd + (lm >> 1);
          uint32_t b0, b1, b2, b3;
          ldsm_x4_t(vb + swz(r, c), b0, b1, b2, b3);
          mma_bf16(o[nd], ph0, ph2, b0, b1);
          mma_bf16(o[nd], pl0, pl2, b0, b1);
          mma_bf16(o[nd + 1], ph0, ph2, b2, b3);
          mma_bf16(o[nd + 1], pl0, pl2, b2, b3);
        }
      }
      __syncthreads();  // the ring slot may be refilled by the next issue()
    }
    cp_async_wait<0>();
  }
  __syncthreads();
  // ---- merge the 4 warps' states per head; lane (qr, qc2) holds head qr, dims 8i + qc2, +1
  lsum += __shfl_xor_sync(0xffffffffu, lsum, 1);
  lsum += __shfl_xor_sync(0xffffffffu, lsum, 2);
  float* st_o = reinterpret_cast<float*>(smem);        // [warps][G][128]
  float* st_m = st_o + kMmaWarps * G * kD;              // [warps][G]
  float* st_l = st_m + kMmaWarps * G;                   // [warps][G]
  if (qr < G) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      st_o[(warp * G + qr) * kD + i * 8 + qc2] = o[i][0];
      st_o[(warp * G + qr) * kD + i * 8 + qc2 + 1] = o[i][1];
    }
    if ((lane & 3) == 0) {
      st_m[warp * G + qr] = m;
      st_l[warp * G + qr] = lsum;
    }
  }
  __syncthreads();
  const int d = tid;  // 128 threads == 128 dims
  for (int j = 0; j < G; ++j) {
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < kMmaWarps; ++w) M = fmaxf(M, st_m[w * G + j]);
    float L = 0.f, O = 0.f;
    if (M != -INFINITY) {
#pragma unroll
      for (int w = 0; w < kMmaWarps; ++w) {
        const float mw = st_m[w * G + j];
        if (mw != -INFINITY) {
          const float c = exp2f(mw - M);
          L = fmaf(st_l[w * G + j], c, L);
          O = fmaf(st_o[(w * G + j) * kD + d], c, O);
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
  // ---- the last CTA of (b, g) merges the splits of its G rows (split order:
  // deterministic) and re-arms the counter for the next call
  __shared__ int s_last;
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = atomicAdd(&counters[bg], 1) == splits - 1;
  __syncthreads();
  if (s_last) {
    __threadfence();
    for (int j = 0; j < G; ++j) {
      const size_t row = (size_t)b * Hq + g * G + j;
      const float* pp = part + row * splits * kPartStride;
      float M = -INFINITY;
      for (int s2 = 0; s2 < splits; ++s2) M = fmaxf(M, __ldcg(pp + s2 * kPartStride));
      float L = 0.f, O = 0.f;
      if (M != -INFINITY) {
        for (int s2 = 0; s2 < splits; ++s2) {
          const float ms = __ldcg(pp + s2 * kPartStride);
          if (ms != -INFINITY) {
            const float c = exp2f(ms - M);
            L = fmaf(__ldcg(pp + s2 * kPartStride + 1), c, L);
            O = fmaf(__ldcg(pp + s2 * kPartStride + 2 + d), c, O);
          }
        }
      }
      store_out(out, out_dtype, row * kD + d, L > 0.f ? O / L : 0.f);
      if (lse_out && d == 0) lse_out[row] = L > 0.f ? (M + log2f(L)) * kLn2 : -INFINITY;
    }
    if (tid == 0) counters[bg] = 0;
  }
}

template <int G>
cudaError_t launch_mma_t(const Geo& g, const sd_paged_kv& kv, const void* q, float scale, float* part, int splits,
                         void* out, float* lse, int* counters, int* err, cudaStream_t st) {
  const int max_tok = ((g.max_seq_len + splits - 1) / splits + 15) & ~15;
  const size_t smem = (size_t)kStagesM * kStageBytesM + sizeof(int) * (max_tok / 16 + 1) + 16;
  static_assert(2 * kStageBytesM >= kMmaWarps * 8 * (kD + 2) * 4, "combine scratch must fit the ring");
  auto kern = attend_rows_mma_kernel<G>;
  cudaError_t e = ensure_dyn_smem(reinterpret_cast<const void*>(kern), smem);
  if (e != cudaSuccess) return e;
  kern<<<dim3(splits, g.B * g.Hkv), kMmaThreads, smem, st>>>(
      reinterpret_cast<const uint16_t*>(q), reinterpret_cast<const char*>(kv.k_pages),
      reinterpret_cast<const char*>(kv.v_pages), kv.page_table, kv.seq_lens, g.max_seq_len, g.max_pages, g.Hkv,
      scale * kLog2e, part, splits, max_tok, out, g.out_dtype, lse, counters, err);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_dense_rows_mma(const Geo& g, const sd_paged_kv& kv, const void* q, float scale, float* part,
                                  int splits, void* out, float* lse, int* counters, int* err, cudaStream_t st) {
  switch (g.G) {
    case 1: return launch_mma_t<1>(g, kv, q, scale, part, splits, out, lse, counters, err, st);
    case 2: return launch_mma_t<2>(g, kv, q, scale, part, splits, out, lse, counters, err, st);
    case 4: return launch_mma_t<4>(g, kv, q, scale, part, splits, out, lse, counters, err, st);
    case 8: return launch_mma_t<8>(g, kv, q, scale, part, splits, out, lse, counters, err, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace sd
