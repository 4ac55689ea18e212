// k_topk.cu - A3 exact top-k over materialised fp32 scores (unfused/debug
// path, per-row fallback of the fused path) and the sequence-shard cut.
//
// Selection rule (P:145 exact oracle top-k; ties toward the smaller token
// index S:200; ascending output S:112): row (b, h) keeps the k_b tokens first
// in the order (score desc, index asc).  Radix select on order-preserving
// uint32 keys finds the exact k-th key and the tie count; one pass in index
// order compacts the winners with block prefix scans (sd_select.cuh).  No
// float atomics anywhere: results are bit-exact and run-to-run identical.
#include "sd_common.cuh"
#include "sd_internal.h"
#include "sd_select.cuh"

namespace sd {
namespace {

constexpr int kTkThreads = 1024;

// k_from: lengths the budget is computed from (global lengths for a sequence
// shard); the selection runs over the local N_b and keeps min(k_b, N_b).
// out_scores (nullable): the selected scores, same order as idx; slots
// [count, k_max) of idx/out_scores are padded with -1 / -inf when pad != 0.
template <int NT>
__global__ void __launch_bounds__(NT) topk_radix_kernel(
    const float* __restrict__ scores, int ld, const int* __restrict__ seq_lens, int max_len,
    const int* __restrict__ k_from, int max_from, int Hq, BudgetDev bud, int* __restrict__ idx,
    int* __restrict__ counts, float* __restrict__ out_scores, int k_max, int pad,
    int* __restrict__ err) {
  __shared__ SelectSmem<NT> sm;
  const int row = blockIdx.x, b = row / Hq, tid = threadIdx.x;
  const int N = seq_len_dev(seq_lens, b, max_len);  // -1: out of range (SEQLEN below)
  const bool regions = !k_from && budget_regions(bud);
  int k, lo = 0, hi = N;
  if (regions) {  // NEXT-1: sinks [0, lo) and locals [hi, N) rank above every score
    const RowBudget rb = row_budget(N, bud);
    k = rb.k;
    lo = rb.lo;
    hi = rb.hi;
  } else {
    const int NK = k_from ? seq_len_dev(k_from, b, max_from) : N;
    k = (NK >= 1 && (bud.k_fixed > 0 || bud.S >= 1.0)) ? budget_k_dev(NK, bud.S, bud.k_fixed) : 0;
    if (k_from) k = NK >= 1 ? min(k, max(N, 0)) : -1;
  }
  int* out = idx + (size_t)row * k_max;
  float* osc = out_scores ? out_scores + (size_t)row * k_max : nullptr;
  if (N < 0 || k < 0 || k > k_max || k > N || (k < 1 && !k_from && !regions) || (!k_from && !regions && bud.k_fixed > N)) {
    if (tid == 0) { set_error(err, SD_DEVERR_SEQLEN); counts[row] = 0; }
    return;
  }
  const float* s = scores + (size_t)row * ld;
  pdl_wait();  // the scores come from the preceding kernel (coherent loads)
  auto key_at = [s, lo, hi](int i) { return (i < lo || i >= hi) ? 0xFFFFFFFFu : score_key(__ldcg(s + i)); };
  uint32_t emitted = 0;
  if (k > 0) {
    uint32_t tau, need_eq;
    radix_select_block<NT>(key_at, N, (uint32_t)k, sm, &tau, &need_eq);
    emitted = emit_block<NT, 4>(key_at, N, tau, need_eq, 0u, sm,
                                        [out, osc](uint32_t pos, int i, uint32_t key) {
                                          out[pos] = i;
                                          if (osc) osc[pos] = key_score(key);
                                        });
  }
  if (pad) {
    for (int j = (int)emitted + tid; j < k_max; j += NT) {
      out[j] = -1;
      if (osc) osc[j] = -INFINITY;
    }
  }
  if (tid == 0) counts[row] = k;
}

// Sequence-shard cut.  all_cand: fp32 [P][rows][k_max]
// candidate scores of every rank in ascending local-index order (-inf pad).
// The global top-k_b over the union is fixed by its k-th key tau and the tie
// count; ties go to lower global index = lower rank, then lower local index.
// Writes this rank's surviving LOCAL indices (ascending) to surv and their
// number to surv_cnt (may be 0).
__global__ void __launch_bounds__(kTkThreads) seqshard_cut_kernel(
    const float* __restrict__ all_cand, const int* __restrict__ cand_idx, int parts, int rank,
    int rows, int Hq, const int* __restrict__ global_seq_lens, double S, int k_fixed, int k_max,
    int* __restrict__ surv, int* __restrict__ surv_cnt, int* __restrict__ err, uint32_t* __restrict__ fbm, int ldw,
    int nw_local) {
  __shared__ SelectSmem<kTkThreads> sm;
  __shared__ uint32_t s_eq_before;
  const int row = blockIdx.x, b = row / Hq, tid = threadIdx.x;
  const int NG = __ldg(global_seq_lens + b);
  const int k = NG >= 1 ? budget_k_dev(NG, S, k_fixed) : 0;
  if (NG < 1 || k < 1 || k > NG || k > k_max) {
    if (tid == 0) { set_error(err, SD_DEVERR_SEQLEN); surv_cnt[row] = 0; }
    return;
  }
  // fbm (optional): the survivors as this rank's selection bitmap row (local tokens)
  uint32_t* fr = fbm ? fbm + (size_t)row * ldw : nullptr;
  if (fr)
    for (int w = tid; w < nw_local; w += kTkThreads) fr[w] = 0u;  // ordered before the bits by the select's barriers
  const int n = parts * k_max;
  auto key_all = [=](int i) {
    const int p = i / k_max, j = i - p * k_max;
    return score_key(__ldg(all_cand + ((size_t)p * rows + row) * k_max + j));
  };
  uint32_t tau, need_eq;
  radix_select_block<kTkThreads>(key_all, n, (uint32_t)k, sm, &tau, &need_eq);
  // ties held by lower ranks come first in global order
  if (tid == 0) s_eq_before = 0;
  __syncthreads();
  uint32_t my_eq = 0;
  for (int i = tid; i < rank * k_max; i += kTkThreads) my_eq += key_all(i) == tau;
  if (my_eq) atomicAdd(&s_eq_before, my_eq);
  __syncthreads();
  const uint32_t eq_before = s_eq_before;
  const float* mine = all_cand + ((size_t)rank * rows + row) * k_max;
  const int* mid = cand_idx + (size_t)row * k_max;
  int* out = surv + (size_t)row * k_max;
  auto key_mine = [mine](int i) { return score_key(__ldg(mine + i)); };
  const uint32_t c = emit_block<kTkThreads, 4>(key_mine, k_max, tau, need_eq, eq_before, sm,
                                               [out, mid, fr](uint32_t pos, int i, uint32_t) {
                                                 const int t = __ldg(mid + i);
                                                 out[pos] = t;
                                                 if (fr) atomicOr(fr + (t >> 5), 1u << (t & 31));
                                               });
  if (tid == 0) surv_cnt[row] = (int)c;
}

}  // namespace

cudaError_t launch_topk(const Geo& g, const float* scores, int ld, const int* seq_lens,
                        Budget bud, int* idx, int* counts, int k_max, int* err, cudaStream_t st) {
  // programmatic dependent launch (the kernel waits before reading the scores)
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(g.B * g.Hq);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cfg.blockDim = dim3(kTkThreads);  // (256-thread CTAs for short rows measured slower: cfg1 38 -> 50 us)
  return cudaLaunchKernelEx(&cfg, topk_radix_kernel<kTkThreads>, scores, ld, seq_lens, g.max_seq_len,
                            (const int*)nullptr, 0, g.Hq, bud.dev(), idx, counts, (float*)nullptr, k_max, 0, err);
}

cudaError_t launch_topk_shard(const Geo& g, const float* scores, int ld, const int* seq_lens,
                              const int* global_lens, int max_global, Budget bud, int* idx, int* counts,
                              float* cand_scores, int k_max, int* err, cudaStream_t st) {
  topk_radix_kernel<kTkThreads><<<g.B * g.Hq, kTkThreads, 0, st>>>(scores, ld, seq_lens, g.max_seq_len, global_lens, max_global,
                                                       g.Hq, bud.dev(),
                                                       idx, counts, cand_scores, k_max, 1,
                                                       err);
  return cudaGetLastError();
}

cudaError_t launch_seqshard_cut(const Geo& g, const float* all_cand, const int* cand_idx, int parts,
                                int rank, const int* global_lens, Budget bud, int k_max, int* surv,
                                int* surv_cnt, int* err, cudaStream_t st, uint32_t* fbm, int ldw) {
  seqshard_cut_kernel<<<g.B * g.Hq, kTkThreads, 0, st>>>(all_cand, cand_idx, parts, rank, g.B * g.Hq,
                                                         g.Hq, global_lens, bud.S, bud.k_fixed, k_max,
                                                         surv, surv_cnt, err, fbm, ldw, (g.max_seq_len + 31) / 32);
  return cudaGetLastError();
}

}  // namespace sd
