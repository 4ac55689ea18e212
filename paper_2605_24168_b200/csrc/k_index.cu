// k_index.cu - A2 indexer scan, materialising fp32 scores (unfused/debug path
// and the per-row fallback of the fused path).  Bandwidth-bound: one 16-B
// coalesced load per token per KV head (C = 8), shared by the G q-heads of
// the group, so the sketch is read exactly once (SURVEY.md 7 hard part 1).
#include "sd_common.cuh"
#include "sd_internal.h"
#include "sd_score.cuh"

namespace sd {
namespace {

constexpr int kScanThreads = 256;
constexpr int kScanTok = 2048;   // tokens per CTA

// grid = (ceil(max_seq_len / kScanTok), B*Hkv)
template <int G, class Sk>
__global__ void __launch_bounds__(kScanThreads) sketch_score_kernel(
    const void* __restrict__ q, int q_dtype, const void* __restrict__ sk,
    const int* __restrict__ channel_ids, int C, const int* __restrict__ page_table,
    const int* __restrict__ seq_lens, int max_len, int max_pages, int Hkv, float* __restrict__ scores, int ld) {
  extern __shared__ float qc[];  // [G][C]
  const int bg = blockIdx.y, b = bg / Hkv, g = bg - b * Hkv;
  const int Hq = Hkv * G;
  const int N = max(0, seq_len_dev(seq_lens, b, max_len));  // invalid rows: not written (topk reports)
  for (int i = threadIdx.x; i < G * C; i += blockDim.x) {
    const int j = i / C, c = i - j * C;
    const int ch = __ldg(channel_ids + ((size_t)b * Hkv + g) * C + c);
    const size_t qe = ((size_t)b * Hq + g * G + j) * kD + ch;
    qc[i] = q_dtype == SD_F32 ? reinterpret_cast<const float*>(q)[qe]
                              : bf_lo(reinterpret_cast<const uint16_t*>(q)[qe]);
  }
  __syncthreads();
  const int* pt = page_table + (size_t)b * max_pages;
  const int tbeg = blockIdx.x * kScanTok;
  const int tend = min(N, tbeg + kScanTok);
  float* srow = scores + ((size_t)b * Hq + g * G) * ld;
  for (int t = tbeg + threadIdx.x; t < tend; t += kScanThreads) {
    const int page = __ldg(pt + (t >> 4));
    const size_t row = sketch_row_elem(page, t & 15, g, Hkv, C);
    float acc[G];
#pragma unroll
    for (int j = 0; j < G; ++j) acc[j] = 0.f;
    for (int c0 = 0; c0 < C; c0 += 8) sketch_fma8<G, Sk>(Sk::load8(sk, row + c0), qc + c0, C, acc);
#pragma unroll
    for (int j = 0; j < G; ++j) srow[(size_t)j * ld + t] = acc[j];
  }
}

// G = 4, C = 8, bf16 sketch: the tensor-core score of sd_score.cuh (the fused
// scan's arithmetic, same MMA placement: 32-token blocks from multiples of 32).
__global__ void __launch_bounds__(kScanThreads) sketch_score_mma_kernel(
    const void* __restrict__ q, int q_dtype, const uint16_t* __restrict__ sk,
    const int* __restrict__ channel_ids, const int* __restrict__ page_table,
    const int* __restrict__ seq_lens, int max_len, int max_pages, int Hkv, float* __restrict__ scores, int ld) {
  constexpr int G = 4, C = 8;
  __shared__ float qc[G * C];
  const int bg = blockIdx.y, b = bg / Hkv, g = bg - b * Hkv;
  const int Hq = Hkv * G;
  const int N = max(0, seq_len_dev(seq_lens, b, max_len));  // invalid rows: not written (topk reports)
  if (threadIdx.x < G * C) {
    const int j = threadIdx.x / C, c = threadIdx.x - j * C;
    const int ch = __ldg(channel_ids + ((size_t)b * Hkv + g) * C + c);
    const size_t qe = ((size_t)b * Hq + g * G + j) * kD + ch;
    qc[threadIdx.x] = q_dtype == SD_F32 ? reinterpret_cast<const float*>(q)[qe]
                                        : bf_lo(reinterpret_cast<const uint16_t*>(q)[qe]);
  }
  __syncthreads();
  const SkMmaQ qm = sk_mma_q([](int j, int c) { return qc[j * C + c]; }, q_dtype == SD_F32 ? 3 : 1);
  const int* pt = page_table + (size_t)b * max_pages;
  const int tbeg = blockIdx.x * kScanTok;
  const int tend = min(N, tbeg + kScanTok);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, u = lane & 3;
  const int tofs = (lane >> 2) + ((u >> 1) << 4), h0 = 2 * (u & 1);
  float* srow = scores + ((size_t)b * Hq + g * G) * ld;
  for (int t0 = tbeg + warp * 32; t0 < tend; t0 += kScanThreads) {
    uint32_t a[4];
    sk_mma_a_global(a, sk, t0, tend,
                    [pt, g, Hkv](int t) { return sketch_row_elem(__ldg(pt + (t >> 4)), t & 15, g, Hkv, C); });
    float d[4];
    sk_mma_score(a, qm, d);
    const int tA = t0 + tofs, tB = tA + 8;
    if (tA < tend) {
      srow[(size_t)h0 * ld + tA] = d[0];
      srow[(size_t)(h0 + 1) * ld + tA] = d[1];
    }
    if (tB < tend) {
      srow[(size_t)h0 * ld + tB] = d[2];
      srow[(size_t)(h0 + 1) * ld + tB] = d[3];
    }
  }
}

// G = 4, C = 8, fp8 e4m3 sketch: the fp8 tensor-core score of sd_score.cuh
// (the fused scan's arithmetic and placement).
__global__ void __launch_bounds__(kScanThreads) sketch_score_mma_f8_kernel(
    const void* __restrict__ q, int q_dtype, const uint8_t* __restrict__ sk,
    const int* __restrict__ channel_ids, const int* __restrict__ page_table,
    const int* __restrict__ seq_lens, int max_len, int max_pages, int Hkv, float* __restrict__ scores, int ld) {
  constexpr int G = 4, C = 8;
  __shared__ float qc[G * C];
  const int bg = blockIdx.y, b = bg / Hkv, g = bg - b * Hkv;
  const int Hq = Hkv * G;
  const int N = max(0, seq_len_dev(seq_lens, b, max_len));  // invalid rows: not written (topk reports)
  if (threadIdx.x < G * C) {
    const int j = threadIdx.x / C, c = threadIdx.x - j * C;
    const int ch = __ldg(channel_ids + ((size_t)b * Hkv + g) * C + c);
    const size_t qe = ((size_t)b * Hq + g * G + j) * kD + ch;
    qc[threadIdx.x] = q_dtype == SD_F32 ? reinterpret_cast<const float*>(q)[qe]
                                        : bf_lo(reinterpret_cast<const uint16_t*>(q)[qe]);
  }
  __syncthreads();
  const SkMmaF8Q qm = sk_mma_q_f8([](int j, int c) { return qc[j * C + c]; });
  const int* pt = page_table + (size_t)b * max_pages;
  const int tbeg = blockIdx.x * kScanTok;
  const int tend = min(N, tbeg + kScanTok);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, u = lane & 3;
  const int tofs = (lane >> 2) + ((u >> 1) << 4), h0 = 2 * (u & 1);
  float* srow = scores + ((size_t)b * Hq + g * G) * ld;
  for (int t0 = tbeg + warp * 32; t0 < tend; t0 += kScanThreads) {
    uint32_t a[4];
    sk_f8_a_global(a, sk, t0, tend,
                   [pt, g, Hkv](int t) { return sketch_row_elem(__ldg(pt + (t >> 4)), t & 15, g, Hkv, C); });
    float d[4];
    sk_mma_score_f8(a, qm, d);
    const int tA = t0 + tofs, tB = tA + 8;
    if (tA < tend) {
      srow[(size_t)h0 * ld + tA] = d[0];
      srow[(size_t)(h0 + 1) * ld + tA] = d[1];
    }
    if (tB < tend) {
      srow[(size_t)h0 * ld + tB] = d[2];
      srow[(size_t)(h0 + 1) * ld + tB] = d[3];
    }
  }
}

// Exact scores from the K pages: one half-warp per token row, kExUnroll rows
// per half-warp in flight (their page ids, then their K rows, are requested
// before any is used), kExTok tokens per CTA so that short rows still spread
// over many SMs (BASELINE cfg1: N = 4096 on 16 CTAs instead of 2).
constexpr int kExUnroll = 4;
constexpr int kExTok = 256;
template <class KV, int G>
__global__ void __launch_bounds__(kScanThreads) exact_score_kernel(
    const void* __restrict__ q, const void* __restrict__ kp, const int* __restrict__ page_table,
    const int* __restrict__ seq_lens, int max_len, int max_pages, int Hkv, float* __restrict__ scores, int ld) {
  const int bg = blockIdx.y, b = bg / Hkv, g = bg - b * Hkv;
  const int Hq = Hkv * G;
  const int N = max(0, seq_len_dev(seq_lens, b, max_len));  // invalid rows: not written (topk reports)
  const int l16 = threadIdx.x & 15, hw = threadIdx.x >> 4;
  constexpr int NHW = kScanThreads / 16;
  float qf[G][8];
#pragma unroll
  for (int j = 0; j < G; ++j) load_q8<KV>(q, ((size_t)b * Hq + g * G + j) * kD + l16 * 8, qf[j]);
  const int* pt = page_table + (size_t)b * max_pages;
  const int tbeg = blockIdx.x * kExTok;
  const int tend = min(N, tbeg + kExTok);
  float* srow = scores + ((size_t)b * Hq + g * G) * ld;
  // uniform trip count per warp: both half-warps iterate together
  for (int t0 = tbeg; t0 < tend; t0 += NHW * kExUnroll) {
    int t[kExUnroll], pg[kExUnroll];
#pragma unroll
    for (int u = 0; u < kExUnroll; ++u) {
      t[u] = t0 + hw + NHW * u;
      pg[u] = __ldg(pt + ((t[u] < tend ? t[u] : tbeg) >> 4));
    }
    typename KV::Raw raw[kExUnroll];
#pragma unroll
    for (int u = 0; u < kExUnroll; ++u)
      raw[u] = KV::load(kp, kv_row_elem(pg[u], (t[u] < tend ? t[u] : tbeg) & 15, g, Hkv) + l16 * 8);
#pragma unroll
    for (int u = 0; u < kExUnroll; ++u) {
      float kf[8];
      KV::unpack(raw[u], kf);
#pragma unroll
      for (int j = 0; j < G; ++j) {
        float s = 0.f;
#pragma unroll
        for (int e = 0; e < 8; ++e) s = fmaf(qf[j][e], kf[e], s);
        s = half_warp_sum(s);
        if (t[u] < tend && l16 == j) srow[(size_t)j * ld + t[u]] = s;
      }
    }
  }
}

template <int G>
cudaError_t index_dispatch(const Geo& g, const sd_paged_kv& kv, const sd_sketch* sk, const void* q,
                           float* scores, int ld, cudaStream_t st) {
  dim3 grid((g.max_seq_len + kScanTok - 1) / kScanTok, g.B * g.Hkv);
  if (sk) {
    const size_t smem = sizeof(float) * G * sk->channels;
    if (sk->dtype == SD_E4M3 && G == 4 && sk->channels == 8)
      sketch_score_mma_f8_kernel<<<grid, kScanThreads, 0, st>>>(
          q, g.kv_dtype, reinterpret_cast<const uint8_t*>(sk->pages), sk->channel_ids, kv.page_table, kv.seq_lens,
          g.max_seq_len, g.max_pages, g.Hkv, scores, ld);
    else if (sk->dtype == SD_E4M3)
      sketch_score_kernel<G, SkE4m3><<<grid, kScanThreads, smem, st>>>(
          q, g.kv_dtype, sk->pages, sk->channel_ids, sk->channels, kv.page_table, kv.seq_lens, g.max_seq_len, g.max_pages, g.Hkv,
          scores, ld);
    else if (G == 4 && sk->channels == 8)
      sketch_score_mma_kernel<<<grid, kScanThreads, 0, st>>>(
          q, g.kv_dtype, reinterpret_cast<const uint16_t*>(sk->pages), sk->channel_ids, kv.page_table, kv.seq_lens,
          g.max_seq_len, g.max_pages, g.Hkv, scores, ld);
    else
      sketch_score_kernel<G, SkBf16><<<grid, kScanThreads, smem, st>>>(
          q, g.kv_dtype, sk->pages, sk->channel_ids, sk->channels, kv.page_table, kv.seq_lens, g.max_seq_len, g.max_pages, g.Hkv,
          scores, ld);
  } else if (g.kv_dtype == SD_BF16) {
    grid.x = (g.max_seq_len + kExTok - 1) / kExTok;
    exact_score_kernel<KvBF16, G><<<grid, kScanThreads, 0, st>>>(q, kv.k_pages, kv.page_table, kv.seq_lens, g.max_seq_len,
                                                                 g.max_pages, g.Hkv, scores, ld);
  } else {
    grid.x = (g.max_seq_len + kExTok - 1) / kExTok;
    exact_score_kernel<KvF32, G><<<grid, kScanThreads, 0, st>>>(q, kv.k_pages, kv.page_table, kv.seq_lens, g.max_seq_len,
                                                                g.max_pages, g.Hkv, scores, ld);
  }
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_index_score(const Geo& g, const sd_paged_kv& kv, const sd_sketch* sk,
                               const void* q, float* scores, int ld, cudaStream_t st) {
  switch (g.G) {
    case 1: return index_dispatch<1>(g, kv, sk, q, scores, ld, st);
    case 2: return index_dispatch<2>(g, kv, sk, q, scores, ld, st);
    case 4: return index_dispatch<4>(g, kv, sk, q, scores, ld, st);
    case 8: return index_dispatch<8>(g, kv, sk, q, scores, ld, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace sd
