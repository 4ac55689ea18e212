// sd_merge.cuh - the split-k LSE merge of one q-row (A5, "flash-decoding
// style" split-k), shared by merge_parts_kernel (k_attend.cu) and
// the GQA-union gather-attend's in-kernel merge (k_attend_pk.cu).
//
// part[row][s] = {m (log2 domain), l, o[128] unnormalised} for split s; one
// thread per output dimension d.  out[row][d] = sum_s 2^(m_s - M) o_s[d] /
// sum_s 2^(m_s - M) l_s with M = max_s m_s, lse = (M + log2 L) ln 2; splits
// merged in split order (deterministic).  Up to kMergeRegSplits splits: every
// split's values in registers after one round of independent L2 loads.
#pragma once
#include "sd_common.cuh"

namespace sd {

constexpr int kMergeRegSplits = 16;   // N <= 128K at 8192 tokens per split
constexpr int kMergeStride = 128 + 2; // == kPartStride (sd_internal.h)

__device__ __forceinline__ void merge_row_regs(const float* __restrict__ part, int splits, int row, int d,
                                               void* __restrict__ out, int out_dtype, float* __restrict__ lse) {
  const float* p = part + (size_t)row * splits * kMergeStride;
  float mv[kMergeRegSplits], lv[kMergeRegSplits], ov[kMergeRegSplits];
  float M = -INFINITY;
#pragma unroll
  for (int s = 0; s < kMergeRegSplits; ++s) {
    const bool in = s < splits;
    mv[s] = in ? __ldcg(p + s * kMergeStride) : -INFINITY;
    lv[s] = in ? __ldcg(p + s * kMergeStride + 1) : 0.f;
    ov[s] = in ? __ldcg(p + s * kMergeStride + 2 + d) : 0.f;
  }
#pragma unroll
  for (int s = 0; s < kMergeRegSplits; ++s) M = fmaxf(M, mv[s]);
  float L = 0.f, O = 0.f;
  if (M != -INFINITY) {
#pragma unroll
    for (int s = 0; s < kMergeRegSplits; ++s) {
      const float c = mv[s] == -INFINITY ? 0.f : exp2f(mv[s] - M);
      L = fmaf(lv[s], c, L);
      O = fmaf(ov[s], c, O);
    }
  }
  store_out(out, out_dtype, (size_t)row * kD + d, L > 0.f ? O / L : 0.f);
  if (lse && d == 0) lse[row] = L > 0.f ? (M + log2f(L)) * kLn2 : -INFINITY;
}

}  // namespace sd
