// sd_internal.h - host-side launchers and workspace layout shared by the
// C-ABI translation unit (sd_api.cu) and the kernel translation units.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "sdattn.h"
#include "sd_sbs.cuh"

namespace sd {

constexpr int kHeadDim = 128;       // the only compiled head_dim
constexpr int kPageSize = 16;       // the only compiled page size
constexpr int kMaxSplits = 64;      // split-k partial slots per (b, h) row (dense / list paths)
constexpr int kPartStride = 128 + 2;  // {m (log2 domain), l, o[128] unnormalised}
constexpr int kScanWarps = 8;         // warps per scan CTA = band regions per 8192-token range
// union-band entries per (b, g, region of 1024 tokens): 512 per head pair (G = 4, the
// tensor-core scan's pair regions), 128 per q-head + 128 for G <= 2 (S = 2 puts ~10% of
// a head's tokens in the band: 95-135 per region at G = 1, measured), every token at G = 8
constexpr int band_region_cap(int G) { return G >= 8 ? 1024 : G == 4 ? 512 : 128 * G + 128; }

// Resolved, validated arguments passed from the C-ABI layer to launchers.
struct Geo {
  int B, Hq, Hkv, G, max_pages, kv_dtype, out_dtype;
  int max_seq_len;
  int sms = 148;  // SM count of the current device (grid sizing)
};

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) at most once per (device,
// kernel, size): the only state the library keeps between calls is this
// per-process cache of an idempotent driver setting (thread-safe).
cudaError_t ensure_dyn_smem(const void* kern, size_t bytes);

struct Budget {
  double S;
  int k_fixed;
  int n_sink = 0, n_local = 0;
  double heavy_fraction = 0.0;
  const int* kfrom = nullptr;  // sequence shard: k_b from these global lengths (<= max_from)
  int max_from = 0;
  BudgetDev dev() const { return BudgetDev{S, k_fixed, n_sink, n_local, heavy_fraction, kfrom, max_from}; }
  bool regions() const { return n_sink != 0 || n_local != 0 || heavy_fraction != 0.0; }
};

// Workspace carve-up; every region is 256-byte aligned.  Computed identically
// by sd_workspace_size and by every entry point.
struct WsLayout {
  size_t err = 0;            // int32 error word (+ reserved)
  size_t part = 0;           // float [B*Hq][part_splits][kPartStride]
  int part_splits = 0;
  size_t scores = 0;         // float [B*Hq][ld]        (budget != NULL)
  int ld = 0;
  size_t idx = 0;            // int32 [B*Hq][k_max]
  size_t counts = 0;         // int32 [B*Hq]
  int k_max = 0;
  // fused path (sample-bracket select, sd_sbs.cuh)
  int nrange = 0, ldw = 0;
  size_t thr = 0;            // uint32 [B*Hq][4]: bracket keys lo, hi; float thresholds flo, fsure
  // band entries (sd_sbs.cuh): union format [B*Hkv][nrange * 8 warps][cap] with G
  // scores each, or (G = 4 tensor-core scan) [B*Hkv][nrange][2 pairs][8 cap] with
  // 2 scores each -- the same bytes
  size_t ent_tok = 0;        // uint32 token | head mask << 24
  size_t ent_sc = 0;         // float scores
  size_t ent_cnt = 0;        // int32 entry count per region (> capacity: overflow -> slow path)
  size_t fbm = 0;            // uint32 [B*Hq][ldw] selection bitmap
  size_t ctr = 0;            // int32 [B*Hkv + 1] last-CTA merge counters + work counter (zero between calls)
  size_t total = 0;
};

WsLayout ws_layout(int B, int Hq, int Hkv, int max_seq_len, bool with_budget, int k_max);

// ---- launchers (return cudaGetLastError()) ---------------------------------
cudaError_t launch_index_score(const Geo& g, const sd_paged_kv& kv, const sd_sketch* sk,
                               const void* q, float* scores, int ld, cudaStream_t st);

cudaError_t launch_topk(const Geo& g, const float* scores, int ld, const int* seq_lens,
                        Budget bud, int* idx, int* counts, int k_max, int* err,
                        cudaStream_t st);

cudaError_t launch_attend_list(const Geo& g, const sd_paged_kv& kv, const void* q,
                               const int* idx, const int* counts, int k_max,
                               const float* weights, float scale, float* part, int splits,
                               int allow_empty, int* err, cudaStream_t st);

cudaError_t launch_topk_shard(const Geo& g, const float* scores, int ld, const int* seq_lens,
                              const int* global_lens, int max_global, Budget bud, int* idx, int* counts,
                              float* cand_scores, int k_max, int* err, cudaStream_t st);

// Per-head index lists (ascending, < N_b; checked per entry like attend_list_kernel: an
// out-of-range / out-of-order entry is skipped with SD_DEVERR_INDEX_RANGE / _ORDER, a count
// outside [1, min(k_max, N_b)] clamped with SD_DEVERR_EMPTY / _SEQLEN) -> selection bitmap
// rows fbm [B*Hq][ldw]; also zeroes *work (the GQA-union attend's item counter).
cudaError_t launch_idx_to_bits(const Geo& g, const int* seq_lens, const int* idx, const int* counts, int k_max,
                               uint32_t* fbm, int ldw, int* work, int* err, cudaStream_t st);
// fbm (nullable): also write the survivors as selection bitmap rows [B*Hq][ldw] over the local tokens
cudaError_t launch_seqshard_cut(const Geo& g, const float* all_cand, const int* cand_idx, int parts,
                                int rank, const int* global_lens, Budget bud, int k_max, int* surv,
                                int* surv_cnt, int* err, cudaStream_t st, uint32_t* fbm = nullptr, int ldw = 0);

// Combine `splits` unnormalised partials per row into out / lse.
cudaError_t launch_merge_parts(const float* part, int rows, int splits, void* out,
                               int out_dtype, float* lse, cudaStream_t st);

// Same, launched as a programmatic dependent of the preceding kernel (PDL).
cudaError_t launch_merge_parts_pdl(const float* part, int rows, int splits, void* out,
                                   int out_dtype, float* lse, cudaStream_t st);

// Combine normalised (o, lse) parts (cross-GPU partials).
cudaError_t launch_lse_merge(int parts, int rows, const float* part_o, const float* part_lse,
                             int out_dtype, void* out, float* lse, cudaStream_t st);

int choose_splits(int rows, int work_per_row, int min_per_split);

// NEXT-2 weighted stochastic selection (k_stoch.cu); mark: [B*Hq][ldw] scratch
cudaError_t launch_stochastic_select(const Geo& g, const float* scores, const float* u, int ld, const int* seq_lens,
                                     int k_det, int n_samples, uint32_t* mark, int ldw, int* idx, float* weights,
                                     int* counts, int k_max, int* err, cudaStream_t st);

// ---- fused sample-bracket select (k_fused.cu) -------------------------------
struct SbsBuffers {
  uint32_t* thr;
  uint32_t* ent_tok;             // scan union-band entries (see sd_sbs.cuh)
  float* ent_sc;
  int* ent_cnt;
  uint32_t* fbm;
  int* counters;                 // [B*Hkv] merge counters, zeroed by the sample kernel
  int ldw;
  float* scratch;                // [B*Hq][ld] fallback scores
  int ld;
  int* counts_out;               // optional [B*Hq]
  int* idx_out;                  // optional [B*Hq][k_max_out]
  int k_max_out;
  int force_fallback;
  int* err;
  cudaEvent_t* ev = nullptr;     // optional: recorded after sample, scan, select (measurement)
};

cudaError_t launch_sbs_select(const Geo& g, const sd_paged_kv& kv, const sd_sketch& sk, const void* q,
                              Budget bud, const SbsBuffers& w, cudaStream_t st);
// sequence shard: selection bitmaps (after launch_sbs_select with bud.kfrom) -> ascending
// candidates + their fp32 scores (G = 4, C = 8, bf16 sketch only)
cudaError_t launch_sbs_emit(const Geo& g, const sd_paged_kv& kv, const sd_sketch& sk, const void* q,
                            const SbsBuffers& w, int* cand_idx, float* cand_scores, int k_max, cudaStream_t st);

// ---- row-list gather-attend (k_rows.cu: fp32 KV on the CUDA cores; k_rows_mma.cu: bf16 dense decode on the tensor cores)
cudaError_t launch_attend_rows(const Geo& g, const sd_paged_kv& kv, const void* q, const uint32_t* fbm, int ldw,
                               float scale, float* part, int splits, cudaStream_t st);
cudaError_t launch_dense_rows(const Geo& g, const sd_paged_kv& kv, const void* q, float scale, float* part,
                              int splits, int* err, cudaStream_t st);
// the bf16 tensor-core dense kernel folds the split merge into their last CTA per (b, g)
// (counters: int32 [B*Hkv], zero between calls)
cudaError_t launch_dense_rows_mma(const Geo& g, const sd_paged_kv& kv, const void* q, float scale, float* part,
                                  int splits, void* out, float* lse, int* counters, int* err, cudaStream_t st);
// persistent variant (k_attend_pk.cu); the split partials are merged by a
// following merge_parts_kernel (PDL)
cudaError_t launch_attend_union_pk(const Geo& g, const sd_paged_kv& kv, const void* q, const uint32_t* fbm, int ldw,
                                   float scale, float* part, void* out, float* lse, int* counters, cudaStream_t st,
                                   cudaEvent_t ev_attend = nullptr);
int choose_row_splits(int groups, int rows_per_group, int resident_per_sm = 3);

}  // namespace sd
