/*
 * sdattn.h - C ABI of the B200 (sm_100a) sparse decode-attention library.
 *
 * The library implements the one data-parallel hot path of arxiv 2605.24168
 * ("extreme sparsity along the context dimension"): for each decode query an
 * indexer scores all N cached keys, an exact top-k keeps k = max(1, ceil(N/S))
 * of them, and exact softmax attention runs over only the gathered K/V rows,
 * so a step moves O(k*d) instead of O(N*d) bytes (Fig. 1a).
 * Citations: "P:n" = line n of the paper text, "S:n" = line n of
 * the companion CPU spec.  DESIGN.md lists every reading taken where
 * the paper is silent.
 *
 * Conventions (all entry points):
 *  - Every call returns sd_status; SD_OK == 0.  Nothing throws across the ABI.
 *  - Tensor arguments are caller-owned DEVICE pointers (the library never
 *    allocates or frees device memory and keeps no pointer after returning),
 *    except the geometry/budget/descriptor structs, which are HOST pointers
 *    read during the call only.
 *  - Scratch comes from a caller-supplied device workspace of at least
 *    sd_workspace_size() bytes, 256-byte aligned.  Word 0 of the workspace is
 *    the device error word (see sd_read_device_error); the caller zeroes the
 *    workspace once (sd_clear_device_error) before first use.
 *  - All work is enqueued asynchronously on `stream` (a cudaStream_t; NULL is
 *    the legacy default stream).  The host never synchronizes except in
 *    sd_read_device_error.  Calls are re-entrant and thread-safe: the only
 *    state kept between calls is a mutex-guarded per-process record of which
 *    (device, kernel) pairs already had their shared-memory limit raised
 *    (an idempotent cudaFuncSetAttribute); all per-call state lives in the
 *    caller's workspace, so concurrent calls need separate workspaces.
 *  - Host-checked argument errors return SD_ERR_INVALID_ARG and launch nothing.
 *  - Supported specialisations (Table 1 geometry; BASELINE.json):
 *    head_dim == 128, page_size == 16, G = Hq/Hkv in {1,2,4,8},
 *    kv/q dtype in {bf16, f32} (kv_dtype == q_dtype), sketch channels C a
 *    multiple of 8 with C <= 128.  Anything else: SD_ERR_UNSUPPORTED.
 *  - seq_lens[b] (N_b) counts the current decode token: the caller appends
 *    the step's K/V row before calling (vLLM convention; reading 10).
 *    Queries and keys arrive already position-encoded.
 */
#ifndef SDATTN_H
#define SDATTN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t sd_status;
enum {
  SD_OK = 0,
  SD_ERR_INVALID_ARG = 1,   /* bad shape / pointer / budget, nothing launched   */
  SD_ERR_UNSUPPORTED = 2,   /* valid but outside the compiled specialisations     */
  SD_ERR_WORKSPACE = 3,     /* workspace NULL, misaligned or too small            */
  SD_ERR_CUDA = 4,          /* a CUDA launch failed (cudaGetLastError)            */
  SD_ERR_DEVICE_CHECK = 5   /* sd_read_device_error found a device-side error     */
};

/* Device error codes written into workspace word 0 (first error wins). */
enum {
  SD_DEVERR_NONE = 0,
  SD_DEVERR_INDEX_RANGE = 1,    /* index >= N_b or < 0; offending row skipped  */
  SD_DEVERR_INDEX_ORDER = 2,    /* indices not strictly increasing            */
  SD_DEVERR_EMPTY = 3,          /* count == 0 for a (b, h) row                */
  SD_DEVERR_WEIGHT = 4,         /* weight <= 0 or non-finite                  */
  SD_DEVERR_SEQLEN = 5,         /* N_b < 1 or > max_seq_len, or k_b > k_max          */
  SD_DEVERR_CAND_OVERFLOW = 6   /* internal: candidate buffer overflow (fell back)    */
};

typedef int32_t sd_dtype;
enum { SD_BF16 = 0, SD_F32 = 1, SD_E4M3 = 2 /* fp8 e4m3: sketch pages only */ };

typedef void* sd_stream; /* cudaStream_t */

/* Geometry of one decode step (Table 1 caption). */
typedef struct {
  int32_t batch;             /* B: decode queries (one per sequence)             */
  int32_t num_q_heads;       /* Hq                                                */
  int32_t num_kv_heads;      /* Hkv; Hq % Hkv == 0, G = Hq/Hkv, q-head h reads    */
                             /*   KV head h / G (contiguous groups)        */
  int32_t head_dim;          /* D (128)                                           */
  int32_t page_size;         /* tokens per page (16)                       */
  int32_t max_pages_per_seq; /* row stride of page_table                          */
  sd_dtype kv_dtype;         /* element type of K/V pages                         */
  sd_dtype q_dtype;          /* element type of q (== kv_dtype)                   */
  sd_dtype out_dtype;        /* element type of out (bf16 or f32)                 */
} sd_geometry;

/* Paged KV cache ("paged KV-cache backend"; "NHD").
 *   k_pages, v_pages : [num_pages][page_size][Hkv][D]  (NHD inside a page)
 *   page_table       : int32 [B][max_pages_per_seq]; token t of sequence b lives
 *                      at (page_table[b][t / page_size], t % page_size)
 *   seq_lens         : int32 [B], 1 <= N_b <= max_seq_len (device)
 *   max_seq_len      : HOST-side upper bound on every N_b (sizes grids and the
 *                      workspace without reading device memory).  Every kernel
 *                      reads N_b against it: a row with N_b < 1 or
 *                      N_b > max_seq_len is treated as empty (nothing is read
 *                      or written for it; out = 0, lse = -inf) and the device
 *                      error word is set to SD_DEVERR_SEQLEN.                   */
typedef struct {
  const void* k_pages;
  const void* v_pages;
  const int32_t* page_table;
  const int32_t* seq_lens;
  int32_t num_pages;
  int32_t max_seq_len;
} sd_paged_kv;

/* Double-Sparsity channel sketch ("8-channel (16-bit) Double Sparsity";
 * S:181-185).
 *   pages       : bf16 [num_pages][Hkv][page_size][C], page p mirrors KV page p;
 *                 row (p, g, s) holds key channels channel_ids[b][g][0..C) of the
 *                 token at (p, s) (head-major inside a page; reading 8)
 *   channel_ids : int32 [B][Hkv][C], strictly increasing, < D
 *   channels    : C
 * Passing a NULL sd_sketch* selects EXACT scores ŝ = <q, K_t> (oracle top-k,
 * P:145).                                                                      */
typedef struct {
  const void* pages;
  const int32_t* channel_ids;
  int32_t channels;
  sd_dtype dtype;  /* SD_BF16 (0, default) or SD_E4M3 (NEXT-4 low-precision sketch,
                      P:301; channels == 8 only); the scores are the same fp32
                      fma chain over the exactly-converted channel values */
} sd_sketch;

/* Sparsity budget ("each query-head attends to 1/S fraction of total
 * tokens").  k_b = max(1, ceil(N_b / sparsity)) evaluated in double
 * precision, or k_fixed when k_fixed > 0 (absolute form; k_fixed > N_b
 * is a device error SD_DEVERR_SEQLEN).  Both fractional fields are doubles, so
 * a budget such as S = 1.3 or heavy_fraction = 0.7 means exactly what the
 * SPEC's double arithmetic gives.
 * Sink + Local + heavy (NEXT-1), active when any of
 * n_sink, n_local, heavy_fraction is non-zero: with lo = min(n_sink, N_b),
 * hi = max(lo, N_b - min(n_local, N_b)), mid = hi - lo, the row keeps every
 * sink [0, lo), every local [hi, N_b) and the top-kh of the middle [lo, hi),
 * kh = min(k_fixed, mid) if k_fixed > 0, else min(mid, floor(heavy_fraction *
 * mid + 1/2)); sparsity is ignored.  AC8: N = 20000, 128 + 128, 0.20 -> 4205
 * rows.  n_sink, n_local >= 0 and 0 <= heavy_fraction <= 1, else INVALID_ARG;
 * the sequence-shard entries return UNSUPPORTED for such budgets. */
typedef struct {
  double sparsity;
  int32_t k_fixed;
  int32_t n_sink;
  int32_t n_local;
  double heavy_fraction;
} sd_budget;

/* ---- host helpers --------------------------------------------------------- */
const char* sd_status_str(sd_status s);
const char* sd_version(void);

/* Rows kept for one sequence of N tokens (with sinks / locals the
 * total sinks + locals + heavy).  INVALID_ARG if S < 1, N < 1, or
 * k_fixed > N in the plain form, or an invalid NEXT-1 field. */
sd_status sd_budget_k(const sd_budget* budget, int32_t N, int32_t* k);

/* Workspace bytes sufficient for EVERY entry point below called with this
 * geometry, budget (NULL = dense/merge only) and max_seq_len. */
sd_status sd_workspace_size(const sd_geometry* geom, const sd_budget* budget,
                            int32_t max_seq_len, size_t* bytes);

/* Same, for an explicit per-row candidate capacity k_max (the sequence-shard
 * entry points, whose k_b comes from the GLOBAL length and may exceed the
 * local max_seq_len). */
sd_status sd_workspace_size_k(const sd_geometry* geom, int32_t max_seq_len,
                              int32_t k_max, size_t* bytes);

/* Zero the device error word (async on stream). */
sd_status sd_clear_device_error(void* ws, sd_stream stream);

/* Synchronize `stream`, read the device error word into *code and return
 * SD_ERR_DEVICE_CHECK if it is non-zero (SD_OK otherwise). */
sd_status sd_read_device_error(const void* ws, int32_t* code, sd_stream stream);

/* Synchronize `stream` and read the workspace statistics words (cumulative
 * since the last sd_clear_device_error): stats[0] = number of (b, h) rows for
 * which sd_sparse_decode_fused left its sample-bracketed fast selection and
 * computed the row on the exact slow path (same result, more time). n <= 8. */
sd_status sd_read_stats(const void* ws, int32_t* stats, int32_t n, sd_stream stream);

/* ---- A2: indexer scan ---------------------
 * scores[b][h][t] = sum_c q[b][h][ch[b][g][c]] * sketch[b][g][t][c]   (sketch)
 *                 = sum_d q[b][h][d] * K[b][t][g][d]                 (sketch == NULL)
 * fp32, UNSCALED (selection is invariant to the positive softmax scale), for
 * t < N_b; entries t >= N_b are not written.  scores: fp32 [B][Hq][ld],
 * ld >= max_seq_len.  The fp32 summation order (c ascending, fma chain) is the
 * same as inside sd_sparse_decode_fused, so both select identical sets. */
sd_status sd_sparse_index_score(const sd_geometry* geom, const sd_paged_kv* kv,
                                const sd_sketch* sketch, const void* q,
                                float* scores, int32_t ld, sd_stream stream);

/* ---- A3: exact top-k (ties to the smaller index S:200; ascending S:112)
 * For every (b, h): idx[b][h][0..k_b) = the k_b tokens first in the order
 * (score descending, index ascending), written in increasing index order;
 * counts[b][h] = k_b.  Slots k_b..k_max-1 are left untouched.
 * scores as produced by sd_sparse_index_score; seq_lens = the N_b (device);
 * k_max >= max_b k_b (computed from max_seq_len).  Bit-exact: equal fp32
 * scores are ordered by index. */
sd_status sd_topk_select(const sd_geometry* geom, const float* scores, int32_t ld,
                         const int32_t* seq_lens, int32_t max_seq_len,
                         const sd_budget* budget, int32_t* idx, int32_t* counts,
                         int32_t k_max, void* ws, size_t ws_bytes, sd_stream stream);

/* ---- NEXT-2: weighted stochastic selection (vAttention stand-in; P:145,
 * P:158 name the method, S:233-241 fix this design) ---------------------------
 * For every (b, h) with N_b tokens, scores fp32 [B][Hq][ld] and u fp32
 * [B][Hq][ld] (one uniform key in [0, 1) per token: the random draw is an
 * input, so that the CPU oracle sees the same draw):
 *   det    = top-k_d by score, k_d = min(k_det, N_b), ties to the lower index, weight 1;
 *   sample = the ns = min(n_samples, N_b - k_d) other tokens with the smallest
 *            u (ties to the lower index), weight (N_b - k_d) / ns (1 when ns
 *            covers the whole remainder);
 * idx[b][h][0..counts) = det U sample in increasing index order, weights the
 * matching weights (feed both to sd_sparse_gather_attend).  k_max >=
 * min(k_det + n_samples, max_seq_len); ws from sd_workspace_size_k(geom,
 * max_seq_len, k_max). */
sd_status sd_stochastic_select(const sd_geometry* geom, const float* scores, int32_t ld,
                               const float* u, const int32_t* seq_lens, int32_t max_seq_len,
                               int32_t k_det, int32_t n_samples, int32_t* idx, float* weights,
                               int32_t* counts, int32_t k_max, void* ws, size_t ws_bytes,
                               sd_stream stream);

/* ---- A4+A5: gather-attend with split-k LSE merge ("weighted attention
 * given sparse index and associated weights") ---------------------
 * For every (b, h) with I = idx[b][h][0..counts[b][h]) and weights w (NULL = 1):
 *   s_i = scale <q_bh, K_i>,  a_i = w_i e^{s_i} / sum_j w_j e^{s_j},
 *   out[b][h] = sum_i a_i V_i  (out_dtype),  lse[b][h] = log sum_j w_j e^{s_j}
 * (lse nullable).  The result is per query head (the paper's per-head index
 * sets).  With unit weights (weights == NULL) and bf16 KV the lists
 * become selection bitmaps and a K/V row chosen by several q-heads of one GQA
 * group is fetched once (the fused path's union gather-attend); weighted or
 * fp32 calls gather per head.  idx entries must be strictly increasing and
 * < N_b; violations set the device error word and the offending index is
 * skipped (either way).  weights: fp32 [B][Hq][k_max]. */
sd_status sd_sparse_gather_attend(const sd_geometry* geom, const sd_paged_kv* kv,
                                  const void* q, const int32_t* idx,
                                  const int32_t* counts, int32_t k_max,
                                  const float* weights, float scale, void* out,
                                  float* lse, void* ws, size_t ws_bytes,
                                  sd_stream stream);

/* ---- A6: fused decode (BASELINE.json north_star) ----------------------------
 * Indexer scan + exact top-k + gather-attend + merge for all (b, h) in one
 * stream-ordered sequence of launches whose scores never round-trip through
 * HBM.  Result identical to sd_sparse_index_score -> sd_topk_select ->
 * attention over the selected rows.  K/V rows selected by several q-heads of
 * one GQA group are fetched once (union gather).  idx_out (int32
 * [B][Hq][k_max_out], ascending) and counts_out ([B][Hq]) are optional
 * (NULL = not written); if idx_out is given, k_max_out >= max_b k_b. */
sd_status sd_sparse_decode_fused(const sd_geometry* geom, const sd_paged_kv* kv,
                                 const sd_sketch* sketch, const void* q,
                                 const sd_budget* budget, float scale, void* out,
                                 float* lse, int32_t* idx_out, int32_t* counts_out,
                                 int32_t k_max_out, void* ws, size_t ws_bytes,
                                 sd_stream stream);

/* sd_sparse_decode_fused with option flags (0 = sd_sparse_decode_fused):
 *   SD_FUSED_FORCE_SLOW_PATH - every row of the sketch-mode selection takes the
 *   exact slow path (all scores recomputed, full radix select): the result is
 *   identical by construction, which the tests check.  Any other bit:
 *   SD_ERR_INVALID_ARG. */
enum { SD_FUSED_FORCE_SLOW_PATH = 1 };
sd_status sd_sparse_decode_fused_ex(const sd_geometry* geom, const sd_paged_kv* kv,
                                    const sd_sketch* sketch, const void* q,
                                    const sd_budget* budget, float scale, void* out,
                                    float* lse, int32_t* idx_out, int32_t* counts_out,
                                    int32_t k_max_out, void* ws, size_t ws_bytes,
                                    uint32_t flags, sd_stream stream);

/* Measurement helper (not for production use): sd_sparse_decode_fused in
 * sketch mode with a CUDA event recorded after each of its kernels; it
 * synchronizes `stream` and writes the kernels' durations in milliseconds to
 * phase_ms[0..n_phases): [0] sample, [1] scan, [2] select, [3] gather-attend,
 * [4] split merge (entries past 5, or of phases the path does not have, are
 * -1).  The events serialise the kernels (no programmatic-dependent-launch
 * overlap), so the sum exceeds the untimed call's duration.  Returns
 * SD_ERR_INVALID_ARG if sketch == NULL. */
sd_status sd_sparse_decode_fused_timed(const sd_geometry* geom, const sd_paged_kv* kv,
                                       const sd_sketch* sketch, const void* q,
                                       const sd_budget* budget, float scale, void* out,
                                       float* lse, void* ws, size_t ws_bytes,
                                       sd_stream stream, float* phase_ms, int32_t n_phases);

/* ---- A7: dense decode (P:59 dense regime, speedup context) -------
 * Full softmax over all N_b rows; each K/V row is loaded once per GQA group. */
sd_status sd_dense_decode(const sd_geometry* geom, const sd_paged_kv* kv,
                          const void* q, float scale, void* out, float* lse,
                          void* ws, size_t ws_bytes, sd_stream stream);

/* ---- LSE merge of normalised partials (flash-decoding identity) -------------
 * part_o: fp32 [parts][rows][D] (each normalised), part_lse: fp32 [parts][rows]
 * (natural log; -inf marks an empty part).  out[r] = sum_p e^{lse_p - lse} o_p,
 * lse[r] = log sum_p e^{lse_p}; parts are combined in index order
 * (deterministic).  lse nullable. */
sd_status sd_lse_merge(int32_t parts, int32_t rows, int32_t D, const float* part_o,
                       const float* part_lse, sd_dtype out_dtype, void* out,
                       float* lse, sd_stream stream);

/* ---- Sequence sharding, called around two all-gathers ------
 * Rank r holds a contiguous token shard of every sequence: local token j of
 * sequence b is global token token_offset[b] + j, with shards ordered by rank.
 * (1) sd_seqshard_local_topk: the local top-min(k_b, N_local) (k_b from the
 *     GLOBAL length global_seq_lens[b]; order (score desc, index asc), ties to the
 *     lower index) listed in increasing LOCAL index: cand_idx int32
 *     [B][Hq][k_max] (unused tail = -1), cand_scores fp32 [B][Hq][k_max] their
 *     indexer scores (unused tail = -inf).  With a bf16 8-channel sketch and
 *     G = 4 the fused selection runs (scores never in HBM); otherwise the scores
 *     are materialised in the workspace and radix-selected.
 * (2) all-gather cand_scores over ranks -> all_cand [P][B][Hq][k_max].
 * (3) sd_seqshard_cut_attend: the global k_b-th element of the P sorted lists
 *     (ties: lower rank first, then lower local position - equal to lower
 *     global index) fixes how many of this rank's candidates survive; attend
 *     over them -> normalised part_o fp32 [B][Hq][D], part_lse fp32 [B][Hq]
 *     (-inf when none survive).  surv_idx (int32 [B][Hq][k_max], nullable)
 *     receives the surviving LOCAL indices in increasing order and surv_counts
 *     (int32 [B][Hq], nullable) their number (may be 0).
 * (4) all-gather partials, sd_lse_merge in rank order. */
sd_status sd_seqshard_local_topk(const sd_geometry* geom, const sd_paged_kv* kv,
                                 const sd_sketch* sketch, const void* q,
                                 const sd_budget* budget,
                                 const int32_t* global_seq_lens,
                                 int32_t max_global_seq_len, float* cand_scores,
                                 int32_t* cand_idx, int32_t k_max, void* ws,
                                 size_t ws_bytes, sd_stream stream);

sd_status sd_seqshard_cut_attend(const sd_geometry* geom, const sd_paged_kv* kv,
                                 const void* q, const sd_budget* budget,
                                 const int32_t* global_seq_lens,
                                 const float* all_cand, const int32_t* cand_idx,
                                 int32_t k_max, int32_t parts, int32_t rank,
                                 float scale, float* part_o, float* part_lse,
                                 int32_t* surv_idx, int32_t* surv_counts,
                                 void* ws, size_t ws_bytes, sd_stream stream);

#ifdef __cplusplus
}
#endif
#endif /* SDATTN_H */
