// k_fused.cu - the fused decode path (A2 + A3 + union build) with scores that
// never round-trip through HBM: "sample-bracket select" (SBS).
//
// The exact top-k_b of a row (ties to the lower index S:200) is found
// without materialising the B*Hq*N scores:
//
//  1. sbs_sample_kernel (grid B*Hkv): score a deterministic page-strided
//     sample of each sequence (every spg-th page, <= 4096 tokens) for the G
//     q-heads of the KV head and take two sample order statistics per head:
//       r_lo = ceil(k f + z sqrt(k f (1-f)) + 1),  r_hi = floor(k f - z sqrt(...))
//     (f = sample fraction, z = 4).  The 22-bit key buckets holding them give
//     tau_lo (bucket floor) <= tau_hi (bucket ceiling) such that, with
//     overwhelming probability, #{key >= tau_lo} >= k_b >= #{key > tau_hi}.
//     When the sample is the whole row (f = 1) the bracket is the 22-bit
//     bucket of the exact k-th key.
//  2. sbs_scan_kernel (grid chunks x B*Hkv): the bandwidth-bound pass.  A
//     producer warp streams the chunk's sketch pages (256 B per page and KV
//     head, head-major layout) into a shared-memory ring with cp.async.bulk;
//     eight consumer warps form the G scores per token (fma chain identical to
//     sd_sparse_index_score) and compare them with tau_lo / tau_hi.  Only
//     candidates (key >= tau_lo, ~3% of tokens) leave the SM, as (key, token)
//     pairs; "sure" tokens (key > tau_hi) are counted.
//  3. sbs_select_kernel (grid B*Hkv): per head, r = k_b - #sure; the exact r-th
//     key of the band (tau_lo <= key <= tau_hi) by an adaptive radix select
//     over the candidates (all G heads per pass), exact ties resolved by
//     sorting the tied token ids.  The selected sets are OR-ed into a shared
//     bitmap and emitted in ascending token order as the GQA union row list
//     (token | head-mask << 24), plus per-head index lists when requested.
//     If any check fails (bracket missed, candidate overflow, too many ties)
//     the CTA computes the exact result for its (b, g) the slow way: all
//     scores (same fp32 code) into scratch, radix select, ordered emission.
//     The result is identical either way; only the time differs.
//
// Deterministic: the union list order is fixed by the bitmap and there are no
// float atomics, so repeated calls are bitwise identical.
#include <limits.h>

#include "sd_common.cuh"
#include "sd_internal.h"
#include "sd_score.cuh"
#include "sd_select.cuh"

namespace sd {
namespace {

constexpr float kBracketZ = 4.0f;
constexpr int kSampleThreads = 512;
constexpr int kSampleSlots = 8;            // sample tokens per thread (cap 4096)
constexpr int kScanConsumers = 8;          // consumer warps
constexpr int kScanThreads = (kScanConsumers + 1) * 32;
constexpr int kScanPages = 512;            // pages (x16 tokens) per scan CTA
constexpr int kScanStageBytes = 16384;     // one ring stage
constexpr int kScanStages = 4;
constexpr int kCandBytes = 32768;          // smem candidate buffer per scan CTA
constexpr int kSelThreads = 512;
constexpr int kBitmapWords = 16384;        // 64 KB: G * window / 32
constexpr int kTieCap = 2048;

__device__ __forceinline__ float load_q_elem(const void* q, int q_dtype, size_t e) {
  return q_dtype == SD_F32 ? reinterpret_cast<const float*>(q)[e]
                           : bf_lo(reinterpret_cast<const uint16_t*>(q)[e]);
}

template <int G>
__device__ __forceinline__ void load_qc(float* qc, const void* q, int q_dtype, const int* channel_ids, int b,
                                        int g, int Hkv, int C, int nthreads) {
  const int Hq = Hkv * G;
  for (int i = threadIdx.x; i < G * C; i += nthreads) {
    const int j = i / C, c = i - j * C;
    const int ch = __ldg(channel_ids + ((size_t)b * Hkv + g) * C + c);
    qc[i] = load_q_elem(q, q_dtype, ((size_t)b * Hq + g * G + j) * kD + ch);
  }
}

template <int G>
__device__ __forceinline__ void token_scores(const uint16_t* __restrict__ sk, const int* pt, int t, int g, int Hkv,
                                             int C, const float* qc, float* acc) {
  const int page = __ldg(pt + (t >> 4));
  const uint16_t* row = sk + sketch_row_elem(page, t & 15, g, Hkv, C);
#pragma unroll
  for (int j = 0; j < G; ++j) acc[j] = 0.f;
  for (int c0 = 0; c0 < C; c0 += 8) sketch_fma8<G>(ldg_nc_v4(row + c0), qc + c0, C, acc);
}

// Warp-level search of a 2048-bin histogram (highest bin = largest keys) for
// the bin holding the r-th largest element; returns (bin, residual rank).
__device__ __forceinline__ void warp_find_bin(const uint32_t* hist, uint32_t r, int* bin_out, uint32_t* res_out) {
  const int lane = threadIdx.x & 31;
  // lane owns bins [2047 - 64*lane - 63, 2047 - 64*lane]
  const int top = 2047 - 64 * lane;
  uint32_t sum = 0;
#pragma unroll 8
  for (int i = 0; i < 64; ++i) sum += hist[top - i];
  uint32_t incl = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  const uint32_t excl = incl - sum;
  const bool mine = excl < r && incl >= r;
  const uint32_t who = __ballot_sync(0xffffffffu, mine);
  const int src = who ? __ffs(who) - 1 : 31;
  int bin = 0;
  uint32_t res = 1;
  if (lane == src) {
    uint32_t above = excl;
    for (int i = 0; i < 64; ++i) {
      const uint32_t c = hist[top - i];
      if (above + c >= r) {
        bin = top - i;
        res = r - above;
        break;
      }
      above += c;
    }
  }
  *bin_out = __shfl_sync(0xffffffffu, bin, src);
  *res_out = __shfl_sync(0xffffffffu, res, src);
}

// --------------------------------------------------------------------------- 1. sample
template <int G>
__global__ void __launch_bounds__(kSampleThreads) sbs_sample_kernel(
    const void* __restrict__ q, int q_dtype, const uint16_t* __restrict__ sk, const int* __restrict__ channel_ids,
    int C, const int* __restrict__ page_table, const int* __restrict__ seq_lens, int max_pages, int Hkv, float S,
    int k_fixed, uint32_t* __restrict__ thr, int* __restrict__ cnt) {
  constexpr int CAP = kSampleThreads * kSampleSlots;
  extern __shared__ __align__(16) unsigned char smem[];
  uint32_t* keys = reinterpret_cast<uint32_t*>(smem);  // [G][CAP]
  uint32_t* hist = keys + G * CAP;                     // [G][2048]
  float* qc = reinterpret_cast<float*>(hist + G * 2048);
  __shared__ int s_bin[G][2];
  __shared__ uint32_t s_res[G][2];
  const int bg = blockIdx.x, b = bg / Hkv, g = bg - b * Hkv;
  const int Hq = Hkv * G;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int N = __ldg(seq_lens + b);
  const int* pt = page_table + (size_t)b * max_pages;
  load_qc<G>(qc, q, q_dtype, channel_ids, b, g, Hkv, C, kSampleThreads);
  for (int i = tid; i < G * 2048; i += kSampleThreads) hist[i] = 0;
  __syncthreads();
  if (N < 1) {
    if (tid < G) cnt[((size_t)b * Hq + g * G + tid) * 4 + 2] = 1;
    return;
  }
  const int k = min(budget_k_dev(N, S, k_fixed), N);
  const int npg = (N + 15) >> 4;
  const int cap_pages = CAP >> 4;
  const int spg = (npg + cap_pages - 1) / cap_pages;  // page stride
  const int ns_pages = (npg + spg - 1) / spg;
  const int n_slots = ns_pages * 16;
  // all loads of this thread first (latency-bound gather of sample pages)
  uint4 raw[kSampleSlots];
  int tt[kSampleSlots];
#pragma unroll
  for (int u = 0; u < kSampleSlots; ++u) {
    const int i = tid + u * kSampleThreads;
    const int t = (i >> 4) * spg * 16 + (i & 15);
    tt[u] = (i < n_slots && t < N) ? t : -1;
    if (tt[u] >= 0) raw[u] = ldg_nc_v4(sk + sketch_row_elem(__ldg(pt + (t >> 4)), t & 15, g, Hkv, C));
  }
#pragma unroll
  for (int u = 0; u < kSampleSlots; ++u) {
    const int i = tid + u * kSampleThreads;
    float acc[G];
#pragma unroll
    for (int j = 0; j < G; ++j) acc[j] = 0.f;
    if (tt[u] >= 0) {
      sketch_fma8<G>(raw[u], qc, C, acc);
      if (C > 8) {
        const int t = tt[u];
        const uint16_t* row = sk + sketch_row_elem(__ldg(pt + (t >> 4)), t & 15, g, Hkv, C);
        for (int c0 = 8; c0 < C; c0 += 8) sketch_fma8<G>(ldg_nc_v4(row + c0), qc + c0, C, acc);
      }
    }
#pragma unroll
    for (int j = 0; j < G; ++j) {
      const uint32_t key = tt[u] >= 0 ? score_key(acc[j]) : 0u;
      if (i < n_slots) keys[j * CAP + i] = key;
      // the top-11-bit digit of float keys is heavily shared: aggregate equal
      // bins within the warp before the shared-memory atomic
      const uint32_t bin = key ? (key >> 21) : 0xFFFFFFFFu;
      const uint32_t peers = __match_any_sync(0xffffffffu, bin);
      if (key && (tid & 31) == __ffs(peers) - 1) atomicAdd(&hist[j * 2048 + bin], (uint32_t)__popc(peers));
    }
  }
  __syncthreads();
  const int last_sampled = (ns_pages - 1) * spg;
  const int n_s = n_slots - ((last_sampled == npg - 1) ? (npg * 16 - N) : 0);
  int r_lo, r_hi;
  if (n_s >= N) {
    r_lo = r_hi = k;
  } else {
    const double f = (double)n_s / (double)N;
    const double mu = (double)k * f, sd = sqrt((double)k * f * (1.0 - f));
    r_lo = (int)ceil(mu + kBracketZ * sd + 1.0);
    r_hi = (int)floor(mu - kBracketZ * sd);
  }
  const uint32_t ra = (uint32_t)min(r_lo, n_s), rb = (uint32_t)max(r_hi, 1);
  // pass 1 (bits 31..21): warp j searches head j for both ranks
  if (warp < G) {
    int bin;
    uint32_t res;
    warp_find_bin(hist + warp * 2048, ra, &bin, &res);
    if ((tid & 31) == 0) { s_bin[warp][0] = bin; s_res[warp][0] = res; }
    warp_find_bin(hist + warp * 2048, rb, &bin, &res);
    if ((tid & 31) == 0) { s_bin[warp][1] = bin; s_res[warp][1] = res; }
  }
  __syncthreads();
  uint32_t tau[G][2];
#pragma unroll 1
  for (int w = 0; w < 2; ++w) {
    // pass 2 (bits 20..10) among keys of the pass-1 bin, for rank w
    for (int i = tid; i < G * 2048; i += kSampleThreads) hist[i] = 0;
    __syncthreads();
    for (int i = tid; i < n_slots; i += kSampleThreads) {
#pragma unroll
      for (int j = 0; j < G; ++j) {
        const uint32_t key = keys[j * CAP + i];
        if ((int)(key >> 21) == s_bin[j][w]) atomicAdd(&hist[j * 2048 + ((key >> 10) & 2047)], 1u);
      }
    }
    __syncthreads();
    if (warp < G) {
      int bin;
      uint32_t res;
      warp_find_bin(hist + warp * 2048, s_res[warp][w], &bin, &res);
      if ((tid & 31) == 0) s_res[warp][w] = (uint32_t)bin;  // reuse: pass-2 bin
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < G; ++j) {
      const uint32_t pre = ((uint32_t)s_bin[j][w] << 21) | (s_res[j][w] << 10);
      tau[j][w] = w == 0 ? pre : (pre | 0x3FFu);  // lo: bucket floor; hi: bucket ceiling
    }
  }
  if (tid < G) {
    const int j = tid;
    uint32_t lo = tau[j][0], hi = tau[j][1];
    if (r_lo > n_s) lo = 0u;         // not enough sample mass: every token is a candidate
    if (r_hi < 1) hi = 0xFFFFFFFFu;  // no token is sure
    const size_t row = (size_t)b * Hq + g * G + j;
    thr[row * 2 + 0] = lo;
    thr[row * 2 + 1] = hi;
    cnt[row * 4 + 0] = 0;  // n_sure
    cnt[row * 4 + 1] = 0;  // n_cand
    cnt[row * 4 + 2] = 0;  // status
  }
  pdl_launch_dependents();
}

// --------------------------------------------------------------------------- 2. scan
// Float thresholds equivalent to the key tests key(s) >= lo and key(s) > hi on
// finite scores (keys <= 0x007FFFFF / >= 0xFF800000 are -inf / +inf / NaN).
__device__ __forceinline__ float thresh_lo(uint32_t lo) {
  if (lo <= 0x007FFFFFu) return -INFINITY;
  if (lo >= 0xFF800000u) return INFINITY;  // no finite score reaches it
  return key_score(lo);
}
__device__ __forceinline__ float thresh_hi(uint32_t hi) {
  if (hi <= 0x007FFFFFu) return -INFINITY;
  if (hi >= 0xFF800000u) return INFINITY;
  if (hi == 0x7FFFFFFFu) hi = 0x7FFFFFFEu;  // no canonical key equals the -0 pattern
  return key_score(hi);
}

__device__ __forceinline__ void cp_async16_zf(void* dst, const void* src, bool valid) {
  const uint32_t d = smem_u32(dst);
  const int n = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(n) : "memory");
}

// two independent fp32 fma's in one FFMA2 (bit-identical to two fmaf)
__device__ __forceinline__ void ffma2(float& a0, float& a1, float x0, float x1, float y) {
  unsigned long long r, a = ((unsigned long long)__float_as_uint(a1) << 32) | __float_as_uint(a0);
  const unsigned long long xx = ((unsigned long long)__float_as_uint(x1) << 32) | __float_as_uint(x0);
  const unsigned long long yy = ((unsigned long long)__float_as_uint(y) << 32) | __float_as_uint(y);
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(xx), "l"(yy), "l"(a));
  a0 = __uint_as_float((uint32_t)r);
  a1 = __uint_as_float((uint32_t)(r >> 32));
}

constexpr int kScanNT = 256;                 // 8 warps
constexpr int kScanStageTok = 1024;          // tokens per stage (C = 8: 16 KB)
constexpr int kScanStagesC = 4;
constexpr int kScanTokCta = 8192;            // tokens per CTA

// C8: sketch width 8 (q channels in registers, one 16-B row per token);
// otherwise generic C (multiple of 8) with the q channels in shared memory.
template <int G, bool C8>
__global__ void __launch_bounds__(kScanNT) sbs_scan_kernel(
    const void* __restrict__ q, int q_dtype, const char* __restrict__ skb, const int* __restrict__ channel_ids,
    int C, const int* __restrict__ page_table, const int* __restrict__ seq_lens, int max_pages, int Hkv,
    const uint32_t* __restrict__ thr, int* __restrict__ cnt, unsigned long long* __restrict__ cand, int cand_cap) {
  constexpr int CCW = kCandBytes / 8 / G / (kScanNT / 32);  // candidate slots per warp per head
  extern __shared__ __align__(128) unsigned char smem[];
  // ring: stages of kScanStageTok tokens x (2C) bytes (C=8: 16 KB)
  const int stage_tok = kScanStageTok * 8 / C;  // C = 8: 1024 tokens = 16 KB per stage
  const int stage_bytes = kScanStageTok * 16;
  unsigned char* ring = smem;
  unsigned long long* cbuf =
      reinterpret_cast<unsigned long long*>(ring + (size_t)kScanStagesC * stage_bytes);  // [G][8 warps][CCW]
  float* qc = reinterpret_cast<float*>(cbuf + G * (kScanNT / 32) * CCW);                 // [G][C]
  __shared__ int s_pages[kScanTokCta / 16];
  __shared__ float s_flo[G];
  __shared__ int s_wcnt[G][kScanNT / 32], s_base[G][kScanNT / 32], s_ovf;

  const int bg = blockIdx.y, b = bg / Hkv, g = bg - b * Hkv;
  const int Hq = Hkv * G;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int N = __ldg(seq_lens + b);
  const int t0 = blockIdx.x * kScanTokCta;
  if (t0 >= N) {
    pdl_launch_dependents();
    return;
  }
  const int t_end = min(N, t0 + kScanTokCta);
  const int ntok = t_end - t0;
  const int npages = (ntok + 15) >> 4;
  const int* pt = page_table + (size_t)b * max_pages;
  for (int i = tid; i < npages; i += kScanNT) s_pages[i] = __ldg(pt + (t0 >> 4) + i);
  load_qc<G>(qc, q, q_dtype, channel_ids, b, g, Hkv, C, kScanNT);
  if (tid == 0) s_ovf = 0;
  __syncthreads();
  const int nst = (ntok + stage_tok - 1) / stage_tok;
  // cp.async issue of stage s: 16-B chunks; token i of the chunk lives at
  // sketch_row(page i/16, slot i%16) and C/8 chunks long
  const int cpt = C >> 3;  // 16-B chunks per token
  auto issue = [&](int s) {
    if (s < nst) {
      unsigned char* st = ring + (size_t)(s % kScanStagesC) * stage_bytes;
      const int nch = stage_tok * cpt;
      for (int qd = tid; qd < nch; qd += kScanNT) {
        const int i = s * stage_tok + qd / cpt;  // chunk-relative token
        const int c = qd - (qd / cpt) * cpt;
        const bool valid = i < ntok;
        const char* src = valid ? skb + (sketch_row_elem(s_pages[i >> 4], i & 15, g, Hkv, C) + c * 8) * 2 : skb;
        cp_async16_zf(st + (size_t)qd * 16, src, valid);
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
#pragma unroll
  for (int s = 0; s < kScanStagesC - 1; ++s) issue(s);

  float qr[G][8];
  if (C8) {
#pragma unroll
    for (int j = 0; j < G; ++j)
#pragma unroll
      for (int c = 0; c < 8; ++c) qr[j][c] = qc[j * 8 + c];
  }
  pdl_wait();  // thresholds come from the sample kernel
  float flo[G];
#pragma unroll
  for (int j = 0; j < G; ++j) {
    const size_t row = (size_t)b * Hq + g * G + j;
    flo[j] = thresh_lo(__ldg(thr + row * 2 + 0));
  }
  const uint32_t lt_mask = (1u << lane) - 1u;
  int wcnt[G];
#pragma unroll
  for (int j = 0; j < G; ++j) wcnt[j] = 0;
  unsigned long long* wreg = cbuf + (size_t)warp * CCW;  // + j * 8 * CCW

  for (int s = 0; s < nst; ++s) {
    issue(s + kScanStagesC - 1);
    asm volatile("cp.async.wait_group %0;" ::"n"(kScanStagesC - 1) : "memory");
    __syncthreads();
    const unsigned char* st = ring + (size_t)(s % kScanStagesC) * stage_bytes;
#pragma unroll 1
    for (int i0 = 0; i0 < stage_tok; i0 += kScanNT) {
      const int i = i0 + tid;                      // token within the stage
      const int tl = s * stage_tok + i;            // chunk-relative token
      const bool valid = i < stage_tok && tl < ntok;
      float acc[G];
#pragma unroll
      for (int j = 0; j < G; ++j) acc[j] = 0.f;
      if (C8) {
        float x[8];
        unpack_bf16x8(*reinterpret_cast<const uint4*>(st + (size_t)(i < stage_tok ? i : 0) * 16), x);
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          if (G == 1) {
            acc[0] = fmaf(qr[0][c], x[c], acc[0]);
          } else {
#pragma unroll
            for (int j = 0; j < G; j += 2) ffma2(acc[j], acc[j + 1], qr[j][c], qr[j + 1][c], x[c]);
          }
        }
      } else if (i < stage_tok) {
        const uint4* src = reinterpret_cast<const uint4*>(st + (size_t)i * 2 * C);
        for (int c0 = 0; c0 < C; c0 += 8) sketch_fma8<G>(src[c0 >> 3], qc + c0, C, acc);
      }
#pragma unroll
      for (int j = 0; j < G; ++j) {
        const bool c = valid && acc[j] >= flo[j];
        const uint32_t bal = __ballot_sync(0xffffffffu, c);
        if (c) {
          const int pos = wcnt[j] + __popc(bal & lt_mask);
          if (pos < CCW)
            wreg[(size_t)j * 8 * CCW + pos] = ((unsigned long long)score_key(acc[j]) << 32) | (unsigned)(t0 + tl);
        }
        wcnt[j] += __popc(bal);
      }
    }
    __syncthreads();  // slot reuse by the next issue()
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  if (lane == 0) {
#pragma unroll
    for (int j = 0; j < G; ++j) {
      s_wcnt[j][warp] = min(wcnt[j], CCW);
      if (wcnt[j] > CCW) s_ovf = 1;
    }
  }
  __syncthreads();
  if (tid < G) {
    const int j = tid;
    const size_t row = (size_t)b * Hq + g * G + j;
    int tot = 0;
    for (int w = 0; w < kScanNT / 32; ++w) tot += s_wcnt[j][w];
    int base = tot ? atomicAdd(&cnt[row * 4 + 1], tot) : 0;
    for (int w = 0; w < kScanNT / 32; ++w) {
      s_base[j][w] = base;
      base += s_wcnt[j][w];
    }
    if (s_ovf) atomicOr(&cnt[row * 4 + 2], 1);
  }
  __syncthreads();
  // copy: warp w copies its own regions
#pragma unroll 1
  for (int j = 0; j < G; ++j) {
    const size_t row = (size_t)b * Hq + g * G + j;
    unsigned long long* dst = cand + row * cand_cap;
    const unsigned long long* srcw = cbuf + ((size_t)j * 8 + warp) * CCW;
    const int n = s_wcnt[j][warp], base = s_base[j][warp];
    for (int i = lane; i < n; i += 32)
      if (base + i < cand_cap) dst[base + i] = srcw[i];
  }
  pdl_launch_dependents();
}

// --------------------------------------------------------------------------- 3. select + union
template <int G>
__global__ void __launch_bounds__(kSelThreads) sbs_select_kernel(
    const void* __restrict__ q, int q_dtype, const uint16_t* __restrict__ sk, const int* __restrict__ channel_ids,
    int C, const int* __restrict__ page_table, const int* __restrict__ seq_lens, int max_pages, int Hkv, float S,
    int k_fixed, const uint32_t* __restrict__ thr, const int* __restrict__ cnt,
    const unsigned long long* __restrict__ cand, int cand_cap, float* __restrict__ scratch, int ld,
    uint32_t* __restrict__ uni, int* __restrict__ uni_cnt, int uni_cap, int* __restrict__ idx_out,
    int* __restrict__ counts_out, int k_max_out, int force_fallback, int* __restrict__ err) {
  extern __shared__ __align__(16) unsigned char smem[];
  uint32_t* bm = reinterpret_cast<uint32_t*>(smem);        // [G][W/32]
  uint32_t* hist = bm + kBitmapWords;                       // [G][2048]
  uint32_t* ties = hist + G * 2048;                         // [kTieCap]
  SelectSmem<kSelThreads>& sm = *reinterpret_cast<SelectSmem<kSelThreads>*>(ties + kTieCap);
  float* qc = reinterpret_cast<float*>(&sm + 1);            // [G][C]
  __shared__ uint32_t s_lo[G], s_hi[G], s_tau[G], s_need[G], s_pre[G], s_eqoff[G];
  __shared__ int s_ncand[G], s_r[G], s_shift[G], s_prev[G], s_done[G], s_cut[G], s_sure[G], s_fb, s_ntie;

  const int bg = blockIdx.x, b = bg / Hkv, g = bg - b * Hkv;
  const int Hq = Hkv * G;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int N = __ldg(seq_lens + b);
  const int* pt = page_table + (size_t)b * max_pages;
  load_qc<G>(qc, q, q_dtype, channel_ids, b, g, Hkv, C, kSelThreads);
  pdl_wait();
  const int k = N >= 1 ? budget_k_dev(N, S, k_fixed) : 0;
  if (N < 1 || k > N) {
    if (tid == 0) {
      set_error(err, SD_DEVERR_SEQLEN);
      uni_cnt[bg] = 0;
    }
    return;
  }
  if (tid == 0) s_fb = force_fallback;
  __syncthreads();
  if (tid < G) {
    const int j = tid;
    const size_t row = (size_t)b * Hq + g * G + j;
    const int n_cand = cnt[row * 4 + 1], status = cnt[row * 4 + 2];
    const uint32_t lo = thr[row * 2 + 0], hi = thr[row * 2 + 1];
    if (status || n_cand > cand_cap || k > n_cand) atomicOr(&s_fb, 1);
    s_lo[j] = lo;
    s_hi[j] = hi;
    s_ncand[j] = min(n_cand, cand_cap);
    s_sure[j] = 0;
    // band offsets off = key - lo lie in [0, hi - lo]; resolve them digit by
    // digit from the top, <= 11 bits per pass
    const uint32_t span = hi - lo;
    const int bits = span ? 32 - __clz(span) : 1;
    s_prev[j] = bits;
    s_shift[j] = bits > 11 ? bits - 11 : 0;
    s_pre[j] = 0;
  }
  for (int i = tid; i < G * 2048; i += kSelThreads) hist[i] = 0;
  __syncthreads();
  // ---- phase A: exact r-th key of each head's band, all heads per pass.
  // Pass 0 also counts the "sure" candidates (key > hi).
  if (!s_fb) {
#pragma unroll 1
    for (int pass = 0; pass < 3; ++pass) {
      if (pass > 0) {
        for (int i = tid; i < G * 2048; i += kSelThreads) hist[i] = 0;
        __syncthreads();
      }
      for (int j = 0; j < G; ++j) {
        if (pass > 0 && s_done[j]) continue;
        const size_t row = (size_t)b * Hq + g * G + j;
        const unsigned long long* cl = cand + row * cand_cap;
        const uint32_t lo = s_lo[j], hi = s_hi[j], pre = s_pre[j];
        const int sh = s_shift[j], prev = s_prev[j];
        const uint32_t dmask = (1u << (prev - sh)) - 1u;
        const int n = s_ncand[j];
        int sure = 0;
        for (int i = tid; i < n; i += kSelThreads) {
          const uint32_t key = (uint32_t)(cl[i] >> 32);
          if (key > hi) {  // sure tokens are not in the band
            ++sure;
            continue;
          }
          const uint32_t off = key - lo;
          if ((uint32_t)((uint64_t)off >> prev) != pre) continue;  // higher digits must match
          atomicAdd(&hist[j * 2048 + ((off >> sh) & dmask)], 1u);
        }
        if (pass == 0) {
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) sure += __shfl_xor_sync(0xffffffffu, sure, o);
          if (lane == 0 && sure) atomicAdd(&s_sure[j], sure);
        }
      }
      __syncthreads();
      if (pass == 0) {
        if (tid < G) {
          const int j = tid;
          const int r = k - s_sure[j];
          s_r[j] = r;
          s_need[j] = (uint32_t)max(r, 0);
          s_done[j] = r <= 0;
          if (r < 0) atomicOr(&s_fb, 1);  // more than k sure tokens: bracket missed
        }
        __syncthreads();
        if (s_fb) break;
      }
      if (warp < G && !s_done[warp]) {
        const int j = warp;
        int bin;
        uint32_t res;
        warp_find_bin(hist + j * 2048, s_need[j], &bin, &res);
        if (lane == 0) {
          const int sh = s_shift[j];
          s_pre[j] = (uint32_t)(((uint64_t)s_pre[j] << (s_prev[j] - sh)) | (uint32_t)bin);
          s_need[j] = res;
          s_prev[j] = sh;
          s_shift[j] = sh > 11 ? sh - 11 : 0;
          s_done[j] = sh == 0;
        }
      }
      __syncthreads();
      bool more = false;
#pragma unroll
      for (int j = 0; j < G; ++j) more |= !s_done[j];
      if (!more) break;
    }
  }
  __syncthreads();
  if (!s_fb) {
    // tau = lo + offset (pre holds the full offset once every digit is fixed)
    if (tid < G) s_tau[tid] = s_r[tid] > 0 ? s_lo[tid] + s_pre[tid] : 0xFFFFFFFFu;
    __syncthreads();
    // exact ties at tau: if fewer are needed than exist, keep the lowest tokens
    for (int j = 0; j < G; ++j) {
      if (s_r[j] <= 0) {
        if (tid == 0) s_cut[j] = INT_MAX;
        continue;
      }
      const size_t row = (size_t)b * Hq + g * G + j;
      const unsigned long long* cl = cand + row * cand_cap;
      if (tid == 0) s_ntie = 0;
      __syncthreads();
      const uint32_t tau = s_tau[j];
      for (int i = tid; i < s_ncand[j]; i += kSelThreads) {
        const unsigned long long e = cl[i];
        if ((uint32_t)(e >> 32) == tau) {
          const int p = atomicAdd(&s_ntie, 1);
          if (p < kTieCap) ties[p] = (uint32_t)e;
        }
      }
      __syncthreads();
      const int ntie = s_ntie;
      if ((uint32_t)ntie > s_need[j]) {
        if (ntie > kTieCap) {
          if (tid == 0) s_fb = 1;
          __syncthreads();
          break;
        }
        int cap2 = 1;
        while (cap2 < ntie) cap2 <<= 1;
        for (int i = ntie + tid; i < cap2; i += kSelThreads) ties[i] = 0xFFFFFFFFu;
        bitonic_sort_smem<kSelThreads>(ties, cap2);
        if (tid == 0) s_cut[j] = (int)ties[s_need[j] - 1];
      } else if (tid == 0) {
        s_cut[j] = INT_MAX;
      }
      __syncthreads();
    }
  }
  __syncthreads();
  const bool fb = s_fb != 0;
  if (fb) {
    // ---- exact generic path for this (b, g): scores into scratch, radix select
    for (int t = tid; t < N; t += kSelThreads) {
      float acc[G];
      token_scores<G>(sk, pt, t, g, Hkv, C, qc, acc);
#pragma unroll
      for (int j = 0; j < G; ++j) scratch[((size_t)b * Hq + g * G + j) * ld + t] = acc[j];
    }
    __syncthreads();
    for (int j = 0; j < G; ++j) {
      const float* sr = scratch + ((size_t)b * Hq + g * G + j) * ld;
      auto key_at = [sr](int i) { return score_key(sr[i]); };
      uint32_t tau, need;
      radix_select_block<kSelThreads>(key_at, N, (uint32_t)k, sm, &tau, &need);
      if (tid == 0) {
        s_tau[j] = tau;
        s_need[j] = need;
        s_eqoff[j] = 0;
      }
    }
    __syncthreads();
  }
  // ---- phase C: windows of W tokens -> bitmap -> ascending union rows
  constexpr int W = kBitmapWords * 32 / G;
  constexpr int WW = W / 32;  // words per head
  uint32_t total_u = 0;
  uint32_t hcount[G];
#pragma unroll
  for (int j = 0; j < G; ++j) hcount[j] = 0;
  uint32_t* ub = uni + (size_t)bg * uni_cap;
  for (int w0 = 0; w0 < N; w0 += W) {
    const int w1 = min(N, w0 + W);
    for (int i = tid; i < kBitmapWords; i += kSelThreads) bm[i] = 0u;
    __syncthreads();
    if (!fb) {
      for (int j = 0; j < G; ++j) {
        const size_t row = (size_t)b * Hq + g * G + j;
        const unsigned long long* cl = cand + row * cand_cap;
        const int n_cand = s_ncand[j];
        const uint32_t hi = s_hi[j], tau = s_tau[j];
        const int r = s_r[j], cut = s_cut[j];
        for (int i = tid; i < n_cand; i += kSelThreads) {
          const unsigned long long e = cl[i];
          const uint32_t key = (uint32_t)(e >> 32);
          const int t = (int)(uint32_t)e;
          if (t < w0 || t >= w1) continue;
          const bool sel = key > hi || (r > 0 && (key > tau || (key == tau && t <= cut)));
          if (sel) atomicOr(&bm[j * WW + ((t - w0) >> 5)], 1u << ((t - w0) & 31));
        }
      }
    } else {
      for (int j = 0; j < G; ++j) {
        const float* sr = scratch + ((size_t)b * Hq + g * G + j) * ld + w0;
        auto key_at = [sr](int i) { return score_key(sr[i]); };
        uint32_t* bmj = bm + j * WW;
        uint32_t eq_seen;
        emit_block<kSelThreads, 4>(key_at, w1 - w0, s_tau[j], s_need[j], s_eqoff[j], sm,
                                   [bmj](uint32_t, int i, uint32_t) { atomicOr(&bmj[i >> 5], 1u << (i & 31)); },
                                   &eq_seen);
        __syncthreads();
        if (tid == 0) s_eqoff[j] += eq_seen;
        __syncthreads();
      }
    }
    __syncthreads();
    // emit union rows (and per-head lists) in ascending token order
    const int nwords = (w1 - w0 + 31) >> 5;
    for (int wb = 0; wb < nwords; wb += kSelThreads) {
      const int wi = wb + tid;
      uint32_t words[G], u = 0;
#pragma unroll
      for (int j = 0; j < G; ++j) {
        words[j] = wi < nwords ? bm[j * WW + wi] : 0u;
        u |= words[j];
      }
      uint32_t tot;
      uint32_t pos = total_u + block_excl_scan<kSelThreads>(__popc(u), sm.warp_tot, &tot);
      uint32_t bits = u;
      while (bits) {
        const int bit = __ffs(bits) - 1;
        bits &= bits - 1;
        uint32_t mask = 0;
#pragma unroll
        for (int j = 0; j < G; ++j) mask |= ((words[j] >> bit) & 1u) << j;
        if (pos < (uint32_t)uni_cap) ub[pos] = (uint32_t)(w0 + wi * 32 + bit) | (mask << 24);
        ++pos;
      }
      total_u += tot;
      if (idx_out) {
#pragma unroll
        for (int j = 0; j < G; ++j) {
          uint32_t tj;
          uint32_t p = hcount[j] + block_excl_scan<kSelThreads>(__popc(words[j]), sm.warp_tot, &tj);
          int* dst = idx_out + ((size_t)b * Hq + g * G + j) * k_max_out;
          uint32_t bj = words[j];
          while (bj) {
            const int bit = __ffs(bj) - 1;
            bj &= bj - 1;
            if (p < (uint32_t)k_max_out) dst[p] = w0 + wi * 32 + bit;
            ++p;
          }
          hcount[j] += tj;
        }
      }
    }
    __syncthreads();
  }
  if (tid == 0) uni_cnt[bg] = (int)min(total_u, (uint32_t)uni_cap);
  if (counts_out && tid < G) counts_out[(size_t)b * Hq + g * G + tid] = k;
  pdl_launch_dependents();
}

template <class Kern>
void set_smem(Kern k, size_t bytes) {
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

template <class Kern, class... Args>
cudaError_t launch_pdl(Kern k, dim3 grid, dim3 block, size_t smem, cudaStream_t st, bool pdl, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, args...);
}

template <int G>
cudaError_t sbs_launch_t(const Geo& geo, const sd_paged_kv& kv, const sd_sketch& skc, const void* q, Budget bud,
                         const SbsBuffers& w, cudaStream_t st) {
  const uint16_t* sk = reinterpret_cast<const uint16_t*>(skc.pages);
  const int C = skc.channels;
  const int BG = geo.B * geo.Hkv;
  cudaError_t e;
  {
    const size_t smem = sizeof(uint32_t) * G * (kSampleThreads * kSampleSlots + 2048) + sizeof(float) * G * C;
    auto kern = sbs_sample_kernel<G>;
    set_smem(kern, smem);
    e = launch_pdl(kern, dim3(BG), dim3(kSampleThreads), smem, st, false, q, geo.kv_dtype, sk, skc.channel_ids, C,
                   kv.page_table, kv.seq_lens, geo.max_pages, geo.Hkv, bud.S, bud.k_fixed, w.thr, w.cnt);
    if (e != cudaSuccess) return e;
  }
  {
    const size_t smem = (size_t)kScanStagesC * kScanStageTok * 16 + kCandBytes + sizeof(float) * G * C;
    dim3 grid((geo.max_seq_len + kScanTokCta - 1) / kScanTokCta, BG);
    if (C == 8) {
      auto kern = sbs_scan_kernel<G, true>;
      set_smem(kern, smem);
      e = launch_pdl(kern, grid, dim3(kScanNT), smem, st, true, q, geo.kv_dtype,
                     reinterpret_cast<const char*>(skc.pages), skc.channel_ids, C, kv.page_table, kv.seq_lens,
                     geo.max_pages, geo.Hkv, (const uint32_t*)w.thr, w.cnt, w.cand, w.cand_cap);
    } else {
      auto kern = sbs_scan_kernel<G, false>;
      set_smem(kern, smem);
      e = launch_pdl(kern, grid, dim3(kScanNT), smem, st, true, q, geo.kv_dtype,
                     reinterpret_cast<const char*>(skc.pages), skc.channel_ids, C, kv.page_table, kv.seq_lens,
                     geo.max_pages, geo.Hkv, (const uint32_t*)w.thr, w.cnt, w.cand, w.cand_cap);
    }
    if (e != cudaSuccess) return e;
  }
  {
    const size_t smem = sizeof(uint32_t) * (kBitmapWords + G * 2048 + kTieCap) + sizeof(SelectSmem<kSelThreads>) +
                        sizeof(float) * G * C;
    auto kern = sbs_select_kernel<G>;
    set_smem(kern, smem);
    e = launch_pdl(kern, dim3(BG), dim3(kSelThreads), smem, st, true, q, geo.kv_dtype, sk, skc.channel_ids, C,
                   kv.page_table, kv.seq_lens, geo.max_pages, geo.Hkv, bud.S, bud.k_fixed, (const uint32_t*)w.thr,
                   (const int*)w.cnt, (const unsigned long long*)w.cand, w.cand_cap, w.scratch, w.ld, w.uni,
                   w.uni_cnt, w.uni_cap, w.idx_out, w.counts_out, w.k_max_out, w.force_fallback, w.err);
  }
  return e;
}

}  // namespace

cudaError_t launch_sbs_select(const Geo& g, const sd_paged_kv& kv, const sd_sketch& sk, const void* q, Budget bud,
                              const SbsBuffers& w, cudaStream_t st) {
  switch (g.G) {
    case 1: return sbs_launch_t<1>(g, kv, sk, q, bud, w, st);
    case 2: return sbs_launch_t<2>(g, kv, sk, q, bud, w, st);
    case 4: return sbs_launch_t<4>(g, kv, sk, q, bud, w, st);
    case 8: return sbs_launch_t<8>(g, kv, sk, q, bud, w, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace sd
