// sd_score.cuh - the A2 indexer score, shared by the unfused scan kernel and
// the fused decode kernels so that both produce bit-identical fp32 scores.
//
// Sketch mode (Double Sparsity):
//   s_hat[t] = sum_{c < C} qc[c] * sk[t][c],  qc[c] = q[h][channel_ids[b][g][c]]
//   evaluated as the fp32 fma chain acc = fma(qc[c], sk[c], acc), c ascending.
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
