// k_stoch.cu - NEXT-2 weighted stochastic index selection (vAttention
// stand-in; P:145, P:158 name the method, S:233-241 fix the design).
//
// Per row (b, h) over its N_b fp32 scores and N_b uniform keys u (an INPUT:
// the random draw is passed in so that the CPU oracle sees the same draw):
//   det    = top-k_d tokens by score (k_d = min(k_det, N_b); ties to the lower
//            index), weight 1;
//   sample = the ns = min(n_samples, N_b - k_d) remainder tokens with the
//            smallest u (ties to the lower index), weight |R| / ns with
//            |R| = N_b - k_d (1 when the whole remainder is taken);
//   output = det U sample in increasing index order with their weights.
// Two radix top-k passes (sd_select.cuh): the first marks det in a bitmap, the
// second selects the top (k_d + ns) of the combined key
//   det -> 0xFFFFFFFF,  remainder -> ~key(u)   (smaller u = larger key),
// so the emission in index order writes det and the sample together.
#include "sd_common.cuh"
#include "sd_internal.h"
#include "sd_select.cuh"

namespace sd {
namespace {

constexpr int kStNT = 1024;

__global__ void __launch_bounds__(kStNT) stochastic_select_kernel(
    const float* __restrict__ scores, const float* __restrict__ u, int ld, const int* __restrict__ seq_lens, int max_len, int Hq,
    int k_det, int n_samples, uint32_t* __restrict__ mark, int ldw, int* __restrict__ idx,
    float* __restrict__ weights, int* __restrict__ counts, int k_max, int* __restrict__ err) {
  __shared__ SelectSmem<kStNT> sm;
  const int row = blockIdx.x, b = row / Hq, tid = threadIdx.x;
  const int N = seq_len_dev(seq_lens, b, max_len);
  if (N < 0) {
    if (tid == 0) {
      set_error(err, SD_DEVERR_SEQLEN);
      counts[row] = 0;
    }
    return;
  }
  const int kd = min(k_det, N), ns = min(n_samples, N - kd), k = kd + ns;
  if (k > k_max) {
    if (tid == 0) {
      set_error(err, SD_DEVERR_SEQLEN);
      counts[row] = 0;
    }
    return;
  }
  const float* s = scores + (size_t)row * ld;
  const float* ur = u + (size_t)row * ld;
  uint32_t* mk = mark + (size_t)row * ldw;
  const int nw = (N + 31) >> 5;
  for (int w = tid; w < nw; w += kStNT) mk[w] = 0u;
  __syncthreads();
  // ---- det = top-k_d by score, marked in the bitmap
  if (kd > 0) {
    auto key1 = [s](int i) { return score_key(__ldg(s + i)); };
    uint32_t tau, need;
    radix_select_block<kStNT>(key1, N, (uint32_t)kd, sm, &tau, &need);
    emit_block<kStNT, 4>(key1, N, tau, need, 0u, sm,
                         [mk](uint32_t, int i, uint32_t) { atomicOr(&mk[i >> 5], 1u << (i & 31)); });
  }
  __threadfence_block();
  __syncthreads();
  if (k == 0) {
    if (tid == 0) counts[row] = 0;
    return;
  }
  // ---- det + the ns smallest-u remainder tokens, emitted in index order
  const float w_s = (ns > 0 && ns < N - kd) ? (float)((double)(N - kd) / (double)ns) : 1.f;
  auto key2 = [mk, ur](int i) {
    return ((mk[i >> 5] >> (i & 31)) & 1u) ? 0xFFFFFFFFu : ~score_key(__ldg(ur + i));
  };
  uint32_t tau2, need2;
  radix_select_block<kStNT>(key2, N, (uint32_t)k, sm, &tau2, &need2);
  int* out = idx + (size_t)row * k_max;
  float* wo = weights + (size_t)row * k_max;
  emit_block<kStNT, 4>(key2, N, tau2, need2, 0u, sm, [out, wo, w_s](uint32_t pos, int i, uint32_t key) {
    out[pos] = i;
    wo[pos] = key == 0xFFFFFFFFu ? 1.f : w_s;
  });
  if (tid == 0) counts[row] = k;
}

}  // namespace

cudaError_t launch_stochastic_select(const Geo& g, const float* scores, const float* u, int ld, const int* seq_lens,
                                     int k_det, int n_samples, uint32_t* mark, int ldw, int* idx, float* weights,
                                     int* counts, int k_max, int* err, cudaStream_t st) {
  stochastic_select_kernel<<<g.B * g.Hq, kStNT, 0, st>>>(scores, u, ld, seq_lens, g.max_seq_len, g.Hq, k_det, n_samples, mark, ldw,
                                                         idx, weights, counts, k_max, err);
  return cudaGetLastError();
}

}  // namespace sd
