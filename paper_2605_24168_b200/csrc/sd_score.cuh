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
#include "sd_common.cuh"

namespace sd {

// Sketch row address (elements) of token (page, slot) for KV head g.
__device__ __forceinline__ size_t sketch_row_elem(int page, int slot, int g, int Hkv, int C) {
  return ((size_t)(page * Hkv + g) * kPS + slot) * C;
}

// One 8-channel chunk of a sketch row -> G partial scores (fma chain continues
// from acc[j]).  qc points at qc[j][c0..c0+8) with row stride C.
template <int G>
__device__ __forceinline__ void sketch_fma8(const uint4& raw, const float* qc, int C, float* acc) {
  float x[8];
  unpack_bf16x8(raw, x);
#pragma unroll
  for (int j = 0; j < G; ++j) {
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[j] = fmaf(qc[j * C + c], x[c], acc[j]);
  }
}

}  // namespace sd
