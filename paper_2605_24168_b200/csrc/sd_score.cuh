// sd_score.cuh - the A2 indexer score, shared by the unfused scan kernel and
// the fused decode kernels so that both produce bit-identical fp32 scores.
//
// Sketch mode (Double Sparsity):
//   s_hat[t] = sum_{c < C} qc[c] * sk[t][c],  qc[c] = q[h][channel_ids[b][g][c]]
//   evaluated as the fp32 fma chain acc = fma(qc[c], sk[c], acc), c ascending,
//   except for G = 4, C = 8, bf16 sketch: one bf16 tensor-core MMA with fp32
//   accumulation (SkMma below), the same in every kernel.
// Exact mode (oracle top-k): s_hat[t] = <q_h, K_t>, evaluated per 16-lane
//   half-warp: lane l sums dims [8l, 8l+8) with an fma chain, then a xor
//   butterfly over 8, 4, 2, 1.
#pragma once
#include <cuda_fp8.h>

#include "sd_common.cuh"

namespace sd {

// Sketch element types (NEXT-4: a lighter indexer).  Both give
// exact fp32 channel values (bf16 and e4m3 embed in fp32), so the score is the
// same fp32 fma chain whatever the storage type.
struct SkBf16 {
  using Raw = uint4;                        // 8 channels
  static constexpr int kBytes = 2;
  __device__ __forceinline__ static Raw load8(const void* base, size_t elem) {
    return ldg_nc_v4(reinterpret_cast<const uint16_t*>(base) + elem);
  }
  __device__ __forceinline__ static void unpack(const Raw& r, float* x) { unpack_bf16x8(r, x); }
};
struct SkE4m3 {
  using Raw = uint2;                        // 8 channels
  static constexpr int kBytes = 1;
  __device__ __forceinline__ static Raw load8(const void* base, size_t elem) {
    return __ldg(reinterpret_cast<const uint2*>(reinterpret_cast<const uint8_t*>(base) + elem));
  }
  __device__ __forceinline__ static void unpack(const Raw& r, float* x) {
    const uint32_t w[2] = {r.x, r.y};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const __nv_fp8x2_storage_t pair = (__nv_fp8x2_storage_t)(w[i >> 1] >> (16 * (i & 1)));
      const __half2_raw h = __nv_cvt_fp8x2_to_halfraw2(pair, __NV_E4M3);
      x[2 * i] = __half2float(__half(__half_raw{h.x}));
      x[2 * i + 1] = __half2float(__half(__half_raw{h.y}));
    }
  }
};

// ---- G = 4 q-heads per KV head, C = 8, bf16 sketch: the score on the tensor
// cores.  The indexer is the contraction [32 tokens x 8 channels] x [8 x 4 heads];
// one mma.sync.m16n8k16 (bf16 in, fp32 accumulate) scores 32 consecutive tokens
// t0 .. t0+31 of one warp for all 4 heads:
//   A (16 x 16, row): A[m][k] = sk[t0 + m][k] (k < 8),  sk[t0 + 16 + m][k - 8] (k >= 8)
//   B (16 x 8, col) : B[k][n] = q[n][k] (k < 8, n < 4),  q[n - 4][k - 8] (k >= 8, n >= 4), else 0
//   D[m][n]         = score(token t0 + m + 16 [n >= 4], head n & 3)
// q (fp32 in general) enters as an exact sum of bf16 parts hi + mid + lo (one
// part when q is bf16), accumulated in that order.  Every kernel that scores
// with this path (fused scan, select fallback, unfused indexer) starts t0 at a
// multiple of 32 and builds the same B, so a (token, head) score is the same
// bits everywhere.  Lane L (r = L/4, u = L%4) holds d[0], d[1] = heads 2(u&1),
// 2(u&1)+1 of token tA = t0 + r + 16(u>>1), and d[2], d[3] = those of tA + 8.
template <int G, class Sk>
struct SkMma {
  static constexpr bool value = false;
};
template <>
struct SkMma<4, SkBf16> {
  static constexpr bool value = true;
};

struct SkMmaQ {
  uint32_t b[3][2];
  int np;
};
__device__ __forceinline__ uint16_t sk_to_bf16(float v) {
  uint16_t h;
  asm("cvt.rn.bf16.f32 %0, %1;" : "=h"(h) : "f"(v));
  return h;
}
// qf(head, channel) -> fp32 q value (0 for heads the caller does not score);
// np = 1 when q is bf16 (exact in one part), else 3.
template <class QF>
__device__ __forceinline__ SkMmaQ sk_mma_q(QF qf, int np) {
  const int lane = threadIdx.x & 31, n = lane >> 2, u = lane & 3;
  const int head = n & 3, grp = n >> 2;
  float v0 = qf(head, 2 * u), v1 = qf(head, 2 * u + 1);
  SkMmaQ r;
  r.np = np;
#pragma unroll
  for (int p = 0; p < 3; ++p) {
    if (p >= np) {  // bf16 q: one exact part
      r.b[p][0] = r.b[p][1] = 0u;
      continue;
    }
    const uint16_t h0 = sk_to_bf16(v0), h1 = sk_to_bf16(v1);
    const uint32_t w = (uint32_t)h0 | ((uint32_t)h1 << 16);
    r.b[p][0] = grp == 0 ? w : 0u;
    r.b[p][1] = grp == 0 ? 0u : w;
    v0 -= __uint_as_float((uint32_t)h0 << 16);  // exact residuals
    v1 -= __uint_as_float((uint32_t)h1 << 16);
  }
  return r;
}
__device__ __forceinline__ void sk_mma(float (&d)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}
__device__ __forceinline__ void sk_mma_score(const uint32_t (&a)[4], const SkMmaQ& q, float (&d)[4]) {
  d[0] = d[1] = d[2] = d[3] = 0.f;
  sk_mma(d, a, q.b[0]);
  if (q.np > 1) {
    sk_mma(d, a, q.b[1]);
    sk_mma(d, a, q.b[2]);
  }
}
// A fragment of tokens t0 .. t0+31 from 16-B rows in shared memory (row i at base + 16 i).
__device__ __forceinline__ void sk_mma_a_smem(uint32_t (&a)[4], uint32_t base) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(a[0]), "=r"(a[1]), "=r"(a[2]), "=r"(a[3])
               : "r"(base + (uint32_t)(threadIdx.x & 31) * 16u));
}
// A fragment from global memory: row(t) -> element offset of token t's sketch
// row (t < n; tokens >= n contribute zero rows).
template <class RowElem>
__device__ __forceinline__ void sk_mma_a_global(uint32_t (&a)[4], const uint16_t* sk, int t0, int n, RowElem row) {
  const int lane = threadIdx.x & 31, r = lane >> 2, u = lane & 3;
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    const int t = t0 + 8 * m + r;
    a[m] = t < n ? __ldg(reinterpret_cast<const uint32_t*>(sk + row(t)) + u) : 0u;
  }
}

// ---- G = 4, C = 8, fp8 e4m3 sketch on the tensor cores (NEXT-4).  The e4m3
// channel values convert exactly to f16 (cvt.rn.f16x2.e4m3x2); the f16 MMA
// (fp32 accumulate) multiplies them with q * 2^s split into two f16 parts
// hi + lo (accumulated in that order), s = 14 - ilogb(max |q| over the group's
// 4 heads x 8 channels), so no part overflows and every q value above 2^-24 of
// that maximum is represented; the result is scaled back by 2^-s (exact).
// Placement (32 tokens t0 .. t0+31, t0 a multiple of 32): A row r holds token
// r (k slots of lanes u = 0, 1) and token r + 16 (u = 2, 3); lane (r, u) reads
// channels 4 (u & 1) .. +3 of its token as ONE 32-bit word (a0 / a2 = its low /
// high channel pairs; a1 / a3 the same for token + 8), B is permuted to match,
// and D is laid out exactly as SkMma's (lane (r, u): heads 2 (u & 1), +1 of
// tokens r + 16 (u >> 1) and + 8).  The same in every kernel that scores an fp8
// sketch with it (fused scan, select slow path, unfused indexer).
template <int G, class Sk>
struct SkMmaF8 {
  static constexpr bool value = false;
};
template <>
struct SkMmaF8<4, SkE4m3> {
  static constexpr bool value = true;
};
struct SkMmaF8Q {
  uint32_t b[2][2];
  float unscale;
};
__device__ __forceinline__ uint32_t f16x2_bits(float lo, float hi) {
  return (uint32_t)__half_as_ushort(__float2half_rn(lo)) | ((uint32_t)__half_as_ushort(__float2half_rn(hi)) << 16);
}
template <class QF>
__device__ __forceinline__ SkMmaF8Q sk_mma_q_f8(QF qf) {
  const int lane = threadIdx.x & 31, n = lane >> 2, u = lane & 3;
  const int head = n & 3, c0 = 4 * (u & 1);
  const bool live = (u >> 1) == (n >> 2);  // the k slots of token group u >> 1 feed columns of group n >> 2
  float v[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) v[i] = qf(head, c0 + i);
  float m = fmaxf(fmaxf(fabsf(v[0]), fabsf(v[1])), fmaxf(fabsf(v[2]), fabsf(v[3])));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  const int sc = m > 0.f ? min(max(14 - ilogbf(m), -120), 120) : 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) v[i] = ldexpf(v[i], sc);
  SkMmaF8Q r;
#pragma unroll
  for (int p = 0; p < 2; ++p) {
    float h[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) h[i] = __half2float(__float2half_rn(v[i]));
    r.b[p][0] = live ? f16x2_bits(v[0], v[1]) : 0u;  // k = 2u, 2u + 1: channels c0, c0 + 1
    r.b[p][1] = live ? f16x2_bits(v[2], v[3]) : 0u;  // k = 2u + 8, 2u + 9: channels c0 + 2, c0 + 3
#pragma unroll
    for (int i = 0; i < 4; ++i) v[i] -= h[i];
  }
  r.unscale = ldexpf(1.f, -sc);
  return r;
}
__device__ __forceinline__ uint32_t f8x2_to_f16x2(uint16_t pair) {
  const __half2_raw h = __nv_cvt_fp8x2_to_halfraw2((__nv_fp8x2_storage_t)pair, __NV_E4M3);
  return (uint32_t)h.x | ((uint32_t)h.y << 16);
}
__device__ __forceinline__ void sk_f8_frag(uint32_t (&a)[4], uint32_t w0, uint32_t w1) {
  a[0] = f8x2_to_f16x2((uint16_t)(w0 & 0xFFFFu));
  a[2] = f8x2_to_f16x2((uint16_t)(w0 >> 16));
  a[1] = f8x2_to_f16x2((uint16_t)(w1 & 0xFFFFu));
  a[3] = f8x2_to_f16x2((uint16_t)(w1 >> 16));
}
__device__ __forceinline__ void sk_mma_f16(float (&d)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}
__device__ __forceinline__ void sk_mma_score_f8(const uint32_t (&a)[4], const SkMmaF8Q& q, float (&d)[4]) {
  d[0] = d[1] = d[2] = d[3] = 0.f;
  sk_mma_f16(d, a, q.b[0]);
  sk_mma_f16(d, a, q.b[1]);
#pragma unroll
  for (int i = 0; i < 4; ++i) d[i] *= q.unscale;
}
// A fragment of tokens t0 .. t0+31 from 8-B e4m3 rows in shared memory (row i at base + 8 i).
__device__ __forceinline__ void sk_f8_a_smem(uint32_t (&a)[4], uint32_t base) {
  const int lane = threadIdx.x & 31, r = lane >> 2, u = lane & 3;
  const uint32_t p = base + (uint32_t)(r + ((u >> 1) << 4)) * 8u + 4u * (u & 1);
  uint32_t w0, w1;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(w0) : "r"(p));
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(w1) : "r"(p + 64u));
  sk_f8_frag(a, w0, w1);
}
// A fragment from global memory: row(t) -> byte offset of token t's 8-B row (t < n).
template <class RowByte>
__device__ __forceinline__ void sk_f8_a_global(uint32_t (&a)[4], const uint8_t* sk, int t0, int n, RowByte row) {
  const int lane = threadIdx.x & 31, r = lane >> 2, u = lane & 3;
  const int ta = t0 + r + ((u >> 1) << 4), tb = ta + 8;
  const uint32_t w0 = ta < n ? __ldg(reinterpret_cast<const uint32_t*>(sk + row(ta)) + (u & 1)) : 0u;
  const uint32_t w1 = tb < n ? __ldg(reinterpret_cast<const uint32_t*>(sk + row(tb)) + (u & 1)) : 0u;
  sk_f8_frag(a, w0, w1);
}

// Sketch row address (elements) of token (page, slot) for KV head g.
__device__ __forceinline__ size_t sketch_row_elem(int page, int slot, int g, int Hkv, int C) {
  return ((size_t)(page * Hkv + g) * kPS + slot) * C;
}

// One 8-channel chunk of a sketch row -> G partial scores (fma chain continues
// from acc[j]).  qc points at qc[j][c0..c0+8) with row stride C.
template <int G, class Sk = SkBf16>
__device__ __forceinline__ void sketch_fma8(const typename Sk::Raw& raw, const float* qc, int C, float* acc) {
  float x[8];
  Sk::unpack(raw, x);
#pragma unroll
  for (int j = 0; j < G; ++j) {
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[j] = fmaf(qc[j * C + c], x[c], acc[j]);
  }
}

}  // namespace sd
