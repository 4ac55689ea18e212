// sd_api.cu - the C ABI (include/sdattn.h): argument validation, budget
// arithmetic, workspace carving and launch sequencing.  No compute happens on
// the host and there is no CPU fallback: every entry point only enqueues
// sm_100a kernels on the caller's stream.
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <utility>

#include "sd_internal.h"

namespace sd {

cudaError_t ensure_dyn_smem(const void* kern, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> done;  // (device, kernel) -> bytes set
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(mu);
  auto it = done.find({dev, kern});
  if (it != done.end() && it->second >= bytes) return cudaSuccess;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) done[{dev, kern}] = bytes;
  return e;
}

static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

WsLayout ws_layout(int B, int Hq, int Hkv, int max_seq_len, bool with_budget, int k_max) {
  WsLayout L;
  size_t off = 256;  // error word + reserved
  const size_t rows = (size_t)B * Hq;
  if (with_budget) L.nrange = (max_seq_len + kRangeTok - 1) / kRangeTok;
  // split partials: the list / dense paths use <= kMaxSplits, the GQA-union attend one per 8192-token range
  L.part_splits = std::max(kMaxSplits, (max_seq_len + kRangeTok - 1) / kRangeTok);
  L.part = off;
  off = align256(off + rows * (size_t)L.part_splits * kPartStride * sizeof(float));
  L.ctr = off;
  off = align256(off + ((size_t)B * Hkv + 1) * sizeof(int));
  if (with_budget) {
    L.ld = (max_seq_len + 63) & ~63;
    L.ldw = L.ld / 32;
    L.k_max = k_max;
    L.scores = off;
    off = align256(off + rows * (size_t)L.ld * sizeof(float));
    L.idx = off;
    off = align256(off + rows * (size_t)k_max * sizeof(int));
    L.counts = off;
    off = align256(off + rows * sizeof(int));
    L.thr = off;  // {lo key, hi key, flo, fsure} per row
    off = align256(off + rows * 4 * sizeof(uint32_t));
    const int G = Hq / Hkv;
    const size_t nreg = (size_t)B * Hkv * L.nrange * kScanWarps;
    const size_t cap = band_region_cap(G);
    const size_t nsub = G == 4 ? 2 : 1;  // the tensor-core scan's per-pair regions (k_fused.cu)
    L.ent_tok = off;
    off = align256(off + nreg * nsub * cap * sizeof(uint32_t));
    L.ent_sc = off;
    off = align256(off + nreg * cap * G * sizeof(float));
    L.ent_cnt = off;
    off = align256(off + nreg * nsub * sizeof(int));
    L.fbm = off;
    off = align256(off + rows * (size_t)L.ldw * sizeof(uint32_t));
  } else {
    // selection bitmaps for sd_sparse_gather_attend's GQA-union path
    L.ld = (max_seq_len + 63) & ~63;
    L.ldw = L.ld / 32;
    L.fbm = off;
    off = align256(off + rows * (size_t)L.ldw * sizeof(uint32_t));
  }
  L.total = off;
  return L;
}

int choose_row_splits(int groups, int rows_per_group, int resident_per_sm) {
  const int target = 148 * resident_per_sm * 5;  // ~5 waves of resident CTAs
  int s = (target + groups - 1) / std::max(groups, 1);
  const int cap = std::max(1, (rows_per_group + 63) / 64);
  s = std::min(s, cap);
  return std::max(1, std::min(s, kMaxSplits));
}

}  // namespace sd

using namespace sd;

namespace {

bool budget_has_regions(const sd_budget* b) {
  return b->n_sink != 0 || b->n_local != 0 || b->heavy_fraction != 0.f;
}

// total selected rows of one sequence (host twin of row_budget, sd_common.cuh)
bool k_from_budget(const sd_budget* b, int N, int* k) {
  if (budget_has_regions(b)) {
    if (N < 0) return false;
    const int lo = std::min(b->n_sink, N), hi = std::max(lo, N - std::min(b->n_local, N));
    const int mid = hi - lo;
    const int kh = b->k_fixed > 0 ? std::min(b->k_fixed, mid)
                                  : std::min(mid, (int)floor((double)b->heavy_fraction * (double)mid + 0.5));
    *k = lo + (N - hi) + kh;
    return true;
  }
  if (b->k_fixed > 0) {
    if (b->k_fixed > N) return false;
    *k = b->k_fixed;
    return true;
  }
  if (!(b->sparsity >= 1.0f)) return false;
  double c = ceil((double)N / (double)b->sparsity);
  *k = c < 1.0 ? 1 : (c > N ? N : (int)c);
  return true;
}

sd_status check_geom(const sd_geometry* g, int max_seq_len, Geo* out) {
  if (!g) return SD_ERR_INVALID_ARG;
  if (g->batch < 1 || g->num_q_heads < 1 || g->num_kv_heads < 1 || g->head_dim < 1 ||
      g->page_size < 1 || g->max_pages_per_seq < 1)
    return SD_ERR_INVALID_ARG;
  if (g->num_q_heads % g->num_kv_heads) return SD_ERR_INVALID_ARG;
  for (int dt : {g->kv_dtype, g->q_dtype, g->out_dtype})
    if (dt != SD_BF16 && dt != SD_F32) return SD_ERR_INVALID_ARG;
  if (max_seq_len < 1 || (long long)max_seq_len > (long long)g->max_pages_per_seq * g->page_size)
    return SD_ERR_INVALID_ARG;
  const int G = g->num_q_heads / g->num_kv_heads;
  if (g->head_dim != kHeadDim || g->page_size != kPageSize) return SD_ERR_UNSUPPORTED;
  if (G != 1 && G != 2 && G != 4 && G != 8) return SD_ERR_UNSUPPORTED;
  if (g->kv_dtype != g->q_dtype) return SD_ERR_UNSUPPORTED;
  out->B = g->batch;
  out->Hq = g->num_q_heads;
  out->Hkv = g->num_kv_heads;
  out->G = G;
  out->max_pages = g->max_pages_per_seq;
  out->kv_dtype = g->kv_dtype;
  out->out_dtype = g->out_dtype;
  out->max_seq_len = max_seq_len;
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) ==
      cudaSuccess && sms > 0)
    out->sms = sms;
  return SD_OK;
}

sd_status check_kv(const sd_paged_kv* kv, bool need_v) {
  if (!kv || !kv->k_pages || !kv->page_table || !kv->seq_lens || kv->num_pages < 1)
    return SD_ERR_INVALID_ARG;
  if (need_v && !kv->v_pages) return SD_ERR_INVALID_ARG;
  return SD_OK;
}

sd_status check_sketch(const sd_sketch* sk) {
  if (!sk) return SD_OK;
  if (!sk->pages || !sk->channel_ids || sk->channels < 1) return SD_ERR_INVALID_ARG;
  if (sk->channels > kHeadDim) return SD_ERR_INVALID_ARG;  // C <= D
  if (sk->channels % 8) return SD_ERR_UNSUPPORTED;
  if (sk->dtype != SD_BF16 && sk->dtype != SD_E4M3) return SD_ERR_INVALID_ARG;
  if (sk->dtype == SD_E4M3 && sk->channels != 8) return SD_ERR_UNSUPPORTED;  // NEXT-4: the 8-channel sketch
  return SD_OK;
}

sd_status check_budget(const sd_budget* b, int max_seq_len, int* k_max) {
  if (!b) return SD_ERR_INVALID_ARG;
  if (b->k_fixed < 0) return SD_ERR_INVALID_ARG;
  if (budget_has_regions(b)) {  // NEXT-1 Sink + Local + heavy
    if (b->n_sink < 0 || b->n_local < 0 || !(b->heavy_fraction >= 0.f && b->heavy_fraction <= 1.f))
      return SD_ERR_INVALID_ARG;
    if (!k_from_budget(b, max_seq_len, k_max)) return SD_ERR_INVALID_ARG;
    *k_max = std::max(*k_max, 1);
    return SD_OK;
  }
  if (b->k_fixed == 0 && !(b->sparsity >= 1.0f)) return SD_ERR_INVALID_ARG;
  if (!k_from_budget(b, max_seq_len, k_max)) return SD_ERR_INVALID_ARG;
  return SD_OK;
}

Budget to_budget(const sd_budget* b) {
  Budget r{b->sparsity, b->k_fixed};
  r.n_sink = b->n_sink;
  r.n_local = b->n_local;
  r.heavy_fraction = b->heavy_fraction;
  return r;
}

sd_status check_ws(const void* ws, size_t ws_bytes, size_t need) {
  if (!ws || ((uintptr_t)ws & 255) || ws_bytes < need) return SD_ERR_WORKSPACE;
  return SD_OK;
}

sd_status cuda_status(cudaError_t e) { return e == cudaSuccess ? SD_OK : SD_ERR_CUDA; }

#define SD_TRY(x)                    \
  do {                               \
    sd_status _s = (x);              \
    if (_s != SD_OK) return _s;      \
  } while (0)
#define SD_CUDA(x)                                  \
  do {                                              \
    if ((x) != cudaSuccess) return SD_ERR_CUDA;     \
  } while (0)

inline char* wsp(void* ws, size_t off) { return reinterpret_cast<char*>(ws) + off; }

}  // namespace

extern "C" {

const char* sd_status_str(sd_status s) {
  switch (s) {
    case SD_OK: return "SD_OK";
    case SD_ERR_INVALID_ARG: return "SD_ERR_INVALID_ARG";
    case SD_ERR_UNSUPPORTED: return "SD_ERR_UNSUPPORTED";
    case SD_ERR_WORKSPACE: return "SD_ERR_WORKSPACE";
    case SD_ERR_CUDA: return "SD_ERR_CUDA";
    case SD_ERR_DEVICE_CHECK: return "SD_ERR_DEVICE_CHECK";
  }
  return "SD_ERR_UNKNOWN";
}

const char* sd_version(void) { return "sdattn 0.1 (sm_100a)"; }

sd_status sd_budget_k(const sd_budget* budget, int32_t N, int32_t* k) {
  if (!budget || !k || N < 1) return SD_ERR_INVALID_ARG;
  int unused;
  SD_TRY(check_budget(budget, N, &unused));
  int kk;
  if (!k_from_budget(budget, N, &kk)) return SD_ERR_INVALID_ARG;
  *k = kk;
  return SD_OK;
}

sd_status sd_workspace_size(const sd_geometry* geom, const sd_budget* budget, int32_t max_seq_len,
                            size_t* bytes) {
  if (!bytes) return SD_ERR_INVALID_ARG;
  Geo g;
  SD_TRY(check_geom(geom, max_seq_len, &g));
  int k_max = 0;
  if (budget) SD_TRY(check_budget(budget, max_seq_len, &k_max));
  *bytes = ws_layout(g.B, g.Hq, g.Hkv, max_seq_len, budget != nullptr, k_max).total;
  return SD_OK;
}

sd_status sd_workspace_size_k(const sd_geometry* geom, int32_t max_seq_len, int32_t k_max, size_t* bytes) {
  if (!bytes || k_max < 1) return SD_ERR_INVALID_ARG;
  Geo g;
  SD_TRY(check_geom(geom, max_seq_len, &g));
  *bytes = ws_layout(g.B, g.Hq, g.Hkv, max_seq_len, true, k_max).total;
  return SD_OK;
}

sd_status sd_clear_device_error(void* ws, sd_stream stream) {
  if (!ws) return SD_ERR_WORKSPACE;
  return cuda_status(cudaMemsetAsync(ws, 0, 256, (cudaStream_t)stream));
}

sd_status sd_read_device_error(const void* ws, int32_t* code, sd_stream stream) {
  if (!ws || !code) return SD_ERR_INVALID_ARG;
  int32_t v = 0;
  SD_CUDA(cudaMemcpyAsync(&v, ws, sizeof(v), cudaMemcpyDeviceToHost, (cudaStream_t)stream));
  SD_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  *code = v;
  return v ? SD_ERR_DEVICE_CHECK : SD_OK;
}

sd_status sd_read_stats(const void* ws, int32_t* stats, int32_t n, sd_stream stream) {
  if (!ws || !stats || n < 1 || n > 8) return SD_ERR_INVALID_ARG;
  SD_CUDA(cudaMemcpyAsync(stats, reinterpret_cast<const int32_t*>(ws) + 1, sizeof(int32_t) * n,
                          cudaMemcpyDeviceToHost, (cudaStream_t)stream));
  SD_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  return SD_OK;
}

sd_status sd_sparse_index_score(const sd_geometry* geom, const sd_paged_kv* kv, const sd_sketch* sketch,
                                const void* q, float* scores, int32_t ld, sd_stream stream) {
  SD_TRY(check_kv(kv, false));
  Geo g;
  SD_TRY(check_geom(geom, kv->max_seq_len, &g));
  SD_TRY(check_sketch(sketch));
  if (!q || !scores || ld < kv->max_seq_len) return SD_ERR_INVALID_ARG;
  return cuda_status(launch_index_score(g, *kv, sketch, q, scores, ld, (cudaStream_t)stream));
}

sd_status sd_topk_select(const sd_geometry* geom, const float* scores, int32_t ld, const int32_t* seq_lens,
                         int32_t max_seq_len, const sd_budget* budget, int32_t* idx, int32_t* counts,
                         int32_t k_max, void* ws, size_t ws_bytes, sd_stream stream) {
  Geo g;
  SD_TRY(check_geom(geom, max_seq_len, &g));
  int kb;
  SD_TRY(check_budget(budget, max_seq_len, &kb));
  if (!scores || !seq_lens || !idx || !counts || ld < max_seq_len || k_max < kb) return SD_ERR_INVALID_ARG;
  SD_TRY(check_ws(ws, ws_bytes, 256));
  const Budget bud = to_budget(budget);
  return cuda_status(launch_topk(g, scores, ld, seq_lens, bud, idx, counts, k_max,
                                 reinterpret_cast<int*>(ws), (cudaStream_t)stream));
}

sd_status sd_stochastic_select(const sd_geometry* geom, const float* scores, int32_t ld, const float* u,
                               const int32_t* seq_lens, int32_t max_seq_len, int32_t k_det, int32_t n_samples,
                               int32_t* idx, float* weights, int32_t* counts, int32_t k_max, void* ws,
                               size_t ws_bytes, sd_stream stream) {
  Geo g;
  SD_TRY(check_geom(geom, max_seq_len, &g));
  if (!scores || !u || !seq_lens || !idx || !weights || !counts || ld < max_seq_len || k_det < 0 || n_samples < 0)
    return SD_ERR_INVALID_ARG;
  if (k_max < 1 || k_max < std::min((long long)k_det + n_samples, (long long)max_seq_len)) return SD_ERR_INVALID_ARG;
  const WsLayout L = ws_layout(g.B, g.Hq, g.Hkv, max_seq_len, true, k_max);
  SD_TRY(check_ws(ws, ws_bytes, L.total));
  return cuda_status(launch_stochastic_select(g, scores, u, ld, seq_lens, k_det, n_samples,
                                              reinterpret_cast<uint32_t*>(wsp(ws, L.fbm)), L.ldw, idx, weights,
                                              counts, k_max, reinterpret_cast<int*>(ws), (cudaStream_t)stream));
}

sd_status sd_sparse_gather_attend(const sd_geometry* geom, const sd_paged_kv* kv, const void* q,
                                  const int32_t* idx, const int32_t* counts, int32_t k_max,
                                  const float* weights, float scale, void* out, float* lse, void* ws,
                                  size_t ws_bytes, sd_stream stream) {
  SD_TRY(check_kv(kv, true));
  Geo g;
  SD_TRY(check_geom(geom, kv->max_seq_len, &g));
  if (!q || !idx || !counts || !out || k_max < 1 || !(scale > 0.f) || !isfinite(scale))
    return SD_ERR_INVALID_ARG;
  const WsLayout L = ws_layout(g.B, g.Hq, g.Hkv, kv->max_seq_len, false, 0);
  SD_TRY(check_ws(ws, ws_bytes, L.total));
  const int rows = g.B * g.Hq;
  float* part = reinterpret_cast<float*>(wsp(ws, L.part));
  cudaStream_t st = (cudaStream_t)stream;
  if (!weights && g.kv_dtype == SD_BF16) {
    // unit weights, bf16 KV: the index lists -> selection bitmaps (same per-entry
    // checks) -> the GQA-union gather-attend: a K/V row selected by several
    // q-heads of a group is fetched once, scored on the tensor cores
    uint32_t* fbm = reinterpret_cast<uint32_t*>(wsp(ws, L.fbm));
    int* ctr = reinterpret_cast<int*>(wsp(ws, L.ctr));
    SD_CUDA(launch_idx_to_bits(g, kv->seq_lens, idx, counts, k_max, fbm, L.ldw, ctr + g.B * g.Hkv,
                               reinterpret_cast<int*>(ws), st));
    return cuda_status(launch_attend_union_pk(g, *kv, q, fbm, L.ldw, scale, part, out, lse, ctr, st, nullptr));
  }
  const int splits = choose_splits(rows, k_max, 64);
  SD_CUDA(launch_attend_list(g, *kv, q, idx, counts, k_max, weights, scale, part, splits, 0,
                             reinterpret_cast<int*>(ws), st));
  return cuda_status(launch_merge_parts(part, rows, splits, out, g.out_dtype, lse, st));
}

namespace {

SbsBuffers sbs_buffers(void* ws, const WsLayout& L) {
  SbsBuffers w;
  w.thr = reinterpret_cast<uint32_t*>(wsp(ws, L.thr));
  w.ent_tok = reinterpret_cast<uint32_t*>(wsp(ws, L.ent_tok));
  w.ent_sc = reinterpret_cast<float*>(wsp(ws, L.ent_sc));
  w.ent_cnt = reinterpret_cast<int*>(wsp(ws, L.ent_cnt));
  w.fbm = reinterpret_cast<uint32_t*>(wsp(ws, L.fbm));
  w.counters = reinterpret_cast<int*>(wsp(ws, L.ctr));
  w.ldw = L.ldw;
  w.scratch = reinterpret_cast<float*>(wsp(ws, L.scores));
  w.ld = L.ld;
  w.counts_out = nullptr;
  w.idx_out = nullptr;
  w.k_max_out = 0;
  w.force_fallback = 0;
  w.err = reinterpret_cast<int*>(ws);
  return w;
}

// The fused step; ev (nullable) = 6 events: [0] before the first kernel, then
// one after each of sample, scan, select, attend, merge (bf16 sketch path).
sd_status fused_impl(const sd_geometry* geom, const sd_paged_kv* kv, const sd_sketch* sketch, const void* q,
                     const sd_budget* budget, float scale, void* out, float* lse, int32_t* idx_out,
                     int32_t* counts_out, int32_t k_max_out, void* ws, size_t ws_bytes, sd_stream stream,
                     cudaEvent_t* ev, uint32_t flags) {
  SD_TRY(check_kv(kv, true));
  Geo g;
  SD_TRY(check_geom(geom, kv->max_seq_len, &g));
  SD_TRY(check_sketch(sketch));
  int k_max;
  SD_TRY(check_budget(budget, kv->max_seq_len, &k_max));
  if (!q || !out || !(scale > 0.f) || !isfinite(scale)) return SD_ERR_INVALID_ARG;
  if (idx_out && k_max_out < k_max) return SD_ERR_INVALID_ARG;
  const WsLayout L = ws_layout(g.B, g.Hq, g.Hkv, kv->max_seq_len, true, k_max);
  SD_TRY(check_ws(ws, ws_bytes, L.total));
  cudaStream_t st = (cudaStream_t)stream;
  int* err = reinterpret_cast<int*>(ws);
  const Budget bud = to_budget(budget);
  const int rows = g.B * g.Hq;
  float* part = reinterpret_cast<float*>(wsp(ws, L.part));
  if (!sketch) {
    // exact-score (oracle top-k) mode: materialised scores + radix top-k
    float* scores = reinterpret_cast<float*>(wsp(ws, L.scores));
    int* idx = idx_out ? idx_out : reinterpret_cast<int*>(wsp(ws, L.idx));
    const int ldi = idx_out ? k_max_out : k_max;
    int* counts = counts_out ? counts_out : reinterpret_cast<int*>(wsp(ws, L.counts));
    SD_CUDA(launch_index_score(g, *kv, nullptr, q, scores, L.ld, st));
    SD_CUDA(launch_topk(g, scores, L.ld, kv->seq_lens, bud, idx, counts, ldi, err, st));
    const int splits = choose_splits(rows, k_max, 64);
    SD_CUDA(launch_attend_list(g, *kv, q, idx, counts, ldi, nullptr, scale, part, splits, 0, err, st));
    return cuda_status(launch_merge_parts(part, rows, splits, out, g.out_dtype, lse, st));
  }
  // sketch (Double Sparsity) mode: sample-bracket select, scores stay on chip
  SbsBuffers w = sbs_buffers(ws, L);
  w.counts_out = counts_out;
  w.idx_out = idx_out;
  w.k_max_out = idx_out ? k_max_out : 0;
  w.force_fallback = (flags & SD_FUSED_FORCE_SLOW_PATH) ? 1 : 0;
  w.err = err;
  w.ev = ev ? ev + 1 : nullptr;
  if (ev) cudaEventRecord(ev[0], st);
  SD_CUDA(launch_sbs_select(g, *kv, *sketch, q, bud, w, st));
  if (g.kv_dtype == SD_BF16)
  {
    // persistent union gather-attend; the split merge is folded into its last CTA per (b, g)
    SD_CUDA(launch_attend_union_pk(g, *kv, q, w.fbm, w.ldw, scale, part, out, lse, w.counters, st,
                                   ev ? ev[4] : nullptr));
    if (ev) cudaEventRecord(ev[5], st);
    return cuda_status(cudaGetLastError());
  }
  const int splits = L.nrange;
  SD_CUDA(launch_attend_rows(g, *kv, q, w.fbm, w.ldw, scale, part, splits, st));
  if (ev) cudaEventRecord(ev[4], st);
  SD_CUDA(launch_merge_parts(part, rows, splits, out, g.out_dtype, lse, st));
  if (ev) cudaEventRecord(ev[5], st);
  return cuda_status(cudaGetLastError());
}

}  // namespace

sd_status sd_sparse_decode_fused(const sd_geometry* geom, const sd_paged_kv* kv, const sd_sketch* sketch,
                                 const void* q, const sd_budget* budget, float scale, void* out, float* lse,
                                 int32_t* idx_out, int32_t* counts_out, int32_t k_max_out, void* ws,
                                 size_t ws_bytes, sd_stream stream) {
  return fused_impl(geom, kv, sketch, q, budget, scale, out, lse, idx_out, counts_out, k_max_out, ws, ws_bytes,
                    stream, nullptr, 0u);
}

sd_status sd_sparse_decode_fused_ex(const sd_geometry* geom, const sd_paged_kv* kv, const sd_sketch* sketch,
                                    const void* q, const sd_budget* budget, float scale, void* out, float* lse,
                                    int32_t* idx_out, int32_t* counts_out, int32_t k_max_out, void* ws,
                                    size_t ws_bytes, uint32_t flags, sd_stream stream) {
  if (flags & ~(uint32_t)SD_FUSED_FORCE_SLOW_PATH) return SD_ERR_INVALID_ARG;
  return fused_impl(geom, kv, sketch, q, budget, scale, out, lse, idx_out, counts_out, k_max_out, ws, ws_bytes,
                    stream, nullptr, flags);
}

sd_status sd_sparse_decode_fused_timed(const sd_geometry* geom, const sd_paged_kv* kv, const sd_sketch* sketch,
                                       const void* q, const sd_budget* budget, float scale, void* out, float* lse,
                                       void* ws, size_t ws_bytes, sd_stream stream, float* phase_ms,
                                       int32_t n_phases) {
  if (!sketch || !phase_ms || n_phases < 1) return SD_ERR_INVALID_ARG;
  cudaEvent_t ev[6];
  for (int i = 0; i < 6; ++i)
    if (cudaEventCreate(&ev[i]) != cudaSuccess) return SD_ERR_CUDA;
  sd_status s = fused_impl(geom, kv, sketch, q, budget, scale, out, lse, nullptr, nullptr, 0, ws, ws_bytes, stream,
                           ev, 0u);
  if (s == SD_OK && cudaStreamSynchronize((cudaStream_t)stream) != cudaSuccess) s = SD_ERR_CUDA;
  for (int i = 0; i < n_phases; ++i) {
    phase_ms[i] = -1.f;
    if (s == SD_OK && i < 5) cudaEventElapsedTime(&phase_ms[i], ev[i], ev[i + 1]);
  }
  for (int i = 0; i < 6; ++i) cudaEventDestroy(ev[i]);
  return s;
}

sd_status sd_dense_decode(const sd_geometry* geom, const sd_paged_kv* kv, const void* q, float scale,
                          void* out, float* lse, void* ws, size_t ws_bytes, sd_stream stream) {
  SD_TRY(check_kv(kv, true));
  Geo g;
  SD_TRY(check_geom(geom, kv->max_seq_len, &g));
  if (!q || !out || !(scale > 0.f) || !isfinite(scale)) return SD_ERR_INVALID_ARG;
  const WsLayout L = ws_layout(g.B, g.Hq, g.Hkv, kv->max_seq_len, false, 0);
  SD_TRY(check_ws(ws, ws_bytes, L.total));
  cudaStream_t st = (cudaStream_t)stream;
  const bool mma = g.kv_dtype == SD_BF16;
  const int splits = choose_row_splits(g.B * g.Hkv, kv->max_seq_len, mma ? 2 : 3);
  float* part = reinterpret_cast<float*>(wsp(ws, L.part));
  if (mma) {
    int* ctr = reinterpret_cast<int*>(wsp(ws, L.ctr));
    SD_CUDA(cudaMemsetAsync(ctr, 0, sizeof(int) * g.B * g.Hkv, st));  // merge counters
    return cuda_status(launch_dense_rows_mma(g, *kv, q, scale, part, splits, out, lse, ctr,
                                             reinterpret_cast<int*>(ws), st));
  }
  SD_CUDA(launch_dense_rows(g, *kv, q, scale, part, splits, reinterpret_cast<int*>(ws), st));
  return cuda_status(launch_merge_parts(part, g.B * g.Hq, splits, out, g.out_dtype, lse, st));
}

sd_status sd_lse_merge(int32_t parts, int32_t rows, int32_t D, const float* part_o, const float* part_lse,
                       sd_dtype out_dtype, void* out, float* lse, sd_stream stream) {
  if (parts < 1 || rows < 1 || !part_o || !part_lse || !out) return SD_ERR_INVALID_ARG;
  if (out_dtype != SD_BF16 && out_dtype != SD_F32) return SD_ERR_INVALID_ARG;
  if (D != kHeadDim) return SD_ERR_UNSUPPORTED;
  return cuda_status(launch_lse_merge(parts, rows, part_o, part_lse, out_dtype, out, lse, (cudaStream_t)stream));
}

sd_status sd_seqshard_local_topk(const sd_geometry* geom, const sd_paged_kv* kv, const sd_sketch* sketch,
                                 const void* q, const sd_budget* budget, const int32_t* global_seq_lens,
                                 int32_t max_global_seq_len, float* cand_scores, int32_t* cand_idx,
                                 int32_t k_max, void* ws, size_t ws_bytes, sd_stream stream) {
  SD_TRY(check_kv(kv, false));
  Geo g;
  SD_TRY(check_geom(geom, kv->max_seq_len, &g));
  SD_TRY(check_sketch(sketch));
  if (budget && budget_has_regions(budget)) return SD_ERR_UNSUPPORTED;  // sinks / locals are global positions
  int kg;
  SD_TRY(check_budget(budget, max_global_seq_len, &kg));
  if (!q || !global_seq_lens || !cand_scores || !cand_idx || k_max < kg ||
      max_global_seq_len < kv->max_seq_len)
    return SD_ERR_INVALID_ARG;
  const WsLayout L = ws_layout(g.B, g.Hq, g.Hkv, kv->max_seq_len, true, k_max);
  SD_TRY(check_ws(ws, ws_bytes, L.total));
  cudaStream_t st = (cudaStream_t)stream;
  int* err = reinterpret_cast<int*>(ws);
  float* scores = reinterpret_cast<float*>(wsp(ws, L.scores));
  int* counts = reinterpret_cast<int*>(wsp(ws, L.counts));
  Budget bud = to_budget(budget);
  if (sketch && g.G == 4 && sketch->channels == 8 && sketch->dtype == SD_BF16) {
    // the fused selection with k_b from the global lengths (scores stay on chip),
    // then the candidates and their scores from the selection bitmaps
    bud.kfrom = global_seq_lens;
    bud.max_from = max_global_seq_len;
    SbsBuffers w = sbs_buffers(ws, L);
    w.counts_out = counts;
    SD_CUDA(launch_sbs_select(g, *kv, *sketch, q, bud, w, st));
    return cuda_status(launch_sbs_emit(g, *kv, *sketch, q, w, cand_idx, cand_scores, k_max, st));
  }
  SD_CUDA(launch_index_score(g, *kv, sketch, q, scores, L.ld, st));
  return cuda_status(launch_topk_shard(g, scores, L.ld, kv->seq_lens, global_seq_lens, max_global_seq_len, bud, cand_idx,
                                       counts, cand_scores, k_max, err, st));
}

sd_status sd_seqshard_cut_attend(const sd_geometry* geom, const sd_paged_kv* kv, const void* q,
                                 const sd_budget* budget, const int32_t* global_seq_lens,
                                 const float* all_cand, const int32_t* cand_idx, int32_t k_max,
                                 int32_t parts, int32_t rank, float scale, float* part_o, float* part_lse,
                                 int32_t* surv_idx, int32_t* surv_counts, void* ws, size_t ws_bytes,
                                 sd_stream stream) {
  SD_TRY(check_kv(kv, true));
  Geo g;
  SD_TRY(check_geom(geom, kv->max_seq_len, &g));
  if (!budget) return SD_ERR_INVALID_ARG;
  if (budget_has_regions(budget)) return SD_ERR_UNSUPPORTED;
  if (budget->k_fixed == 0 && !(budget->sparsity >= 1.0f)) return SD_ERR_INVALID_ARG;
  if (!q || !global_seq_lens || !all_cand || !cand_idx || !part_o || !part_lse || k_max < 1 || parts < 1 ||
      rank < 0 || rank >= parts || !(scale > 0.f))
    return SD_ERR_INVALID_ARG;
  const WsLayout L = ws_layout(g.B, g.Hq, g.Hkv, kv->max_seq_len, true, k_max);
  SD_TRY(check_ws(ws, ws_bytes, L.total));
  cudaStream_t st = (cudaStream_t)stream;
  int* err = reinterpret_cast<int*>(ws);
  int* surv = surv_idx ? surv_idx : reinterpret_cast<int*>(wsp(ws, L.idx));
  int* surv_cnt = surv_counts ? surv_counts : reinterpret_cast<int*>(wsp(ws, L.counts));
  const Budget bud = to_budget(budget);
  const int rows = g.B * g.Hq;
  float* part = reinterpret_cast<float*>(wsp(ws, L.part));
  if (g.kv_dtype == SD_BF16) {
    // survivors -> selection bitmap rows -> the GQA-union gather-attend (each
    // K/V row fetched once per group) -> normalised (o, lse) per row
    uint32_t* fbm = reinterpret_cast<uint32_t*>(wsp(ws, L.fbm));
    int* ctr = reinterpret_cast<int*>(wsp(ws, L.ctr));
    SD_CUDA(launch_seqshard_cut(g, all_cand, cand_idx, parts, rank, global_seq_lens, bud, k_max, surv, surv_cnt,
                                err, st, fbm, L.ldw));
    SD_CUDA(cudaMemsetAsync(ctr + g.B * g.Hkv, 0, sizeof(int), st));  // the attend's work counter
    Geo gf = g;
    gf.out_dtype = SD_F32;
    return cuda_status(launch_attend_union_pk(gf, *kv, q, fbm, L.ldw, scale, part, part_o, part_lse, ctr, st,
                                              nullptr));
  }
  SD_CUDA(launch_seqshard_cut(g, all_cand, cand_idx, parts, rank, global_seq_lens, bud, k_max, surv,
                              surv_cnt, err, st));
  const int splits = choose_splits(rows, k_max, 64);
  SD_CUDA(launch_attend_list(g, *kv, q, surv, surv_cnt, k_max, nullptr, scale, part, splits, 1, err, st));
  // normalised (o, lse) per row for the cross-rank merge
  SD_CUDA(launch_merge_parts(part, rows, splits, part_o, SD_F32, part_lse, st));
  return SD_OK;
}

}  // extern "C"
