// k_fused.cu - the fused decode path, A2 + A3 with scores that never
// round-trip through HBM: "sample-bracket select" (SBS).  The selection is
// consumed by the gather-attend kernels through the contract in sd_sbs.cuh.
//
// The exact top-k_b of a row (ties to the lower index S:200) is found
// without materialising the B*Hq*N scores:
//
//  1. sbs_sample_kernel (grid B*Hkv): score a deterministic page-strided
//     sample of each sequence (every spg-th page, <= 4096 tokens) for the G
//     q-heads of the KV head and take two sample order statistics per head,
//       r_lo = ceil(k f + z sqrt(k f (1-f)) + 1),  r_hi = floor(k f - z sqrt(...))
//     (f = sample fraction, z = 4), located with an 11 + 8 bit histogram.  The
//     floor / ceiling of their 19-bit key bins give tau_lo <= tau_hi such that,
//     with overwhelming probability, #{key >= tau_lo} >= k_b >= #{key > tau_hi}.
//     When the sample is the whole row the bracket is the bin of the exact k-th key.
//  2. sbs_scan_kernel (grid chunks x B*Hkv): the bandwidth-bound pass.  The
//     chunk's sketch rows (16 B per token and KV head) stream through a
//     3-stage cp.async ring; each token's G scores are formed with the same
//     fp32 fma chain as sd_sparse_index_score (packed FFMA2).  Tokens above
//     tau_hi ("sure") go straight into the selection bitmap fbm; tokens inside
//     the bracket ("band") are appended with their G scores to the warp's region.
//  3. sbs_select_kernel (grid B*Hq, one CTA per q-head): sure = popcount of the
//     row's bitmap, r = k_b - sure; the exact r-th largest band key tau is found
//     by an adaptive radix select over the head's band entries, exact ties at
//     tau kept lowest token first, and the band winners OR-ed into fbm.  If a
//     check fails (bracket missed, too many candidates, too many ties) the CTA
//     computes the row exactly the slow way (all scores, same fp32 code, radix
//     select, ordered emission) into the same fbm.  Identical result either way.
//
// Deterministic: no float atomics; union rows are rebuilt in token order.
#include <limits.h>
#include <stdlib.h>
#include <math.h>

#include <algorithm>
#include <type_traits>

#include "sd_common.cuh"
#include "sd_internal.h"
#include "sd_sbs.cuh"
#include "sd_score.cuh"
#include "sd_select.cuh"

namespace sd {
namespace {

constexpr float kBracketZ = 4.0f;
constexpr int kSampleThreads = 1024;      // sample CTA (one per (b, g)): 4096-token sample, 1 CTA/SM
constexpr int kSampleSlots = 4;            // sample tokens per thread
// More (b, g) rows than SMs and sequences up to 80K tokens: 512-thread CTAs
// (2048-token sample, 2 CTAs/SM), one wave instead of two.  Longer sequences
// keep the 4096-token sample: the bracket (and the select's band) widens as
// sqrt(k N / sample) and costs more than the second sample wave (cfg4 turn 66:
// 376 vs 389 us).
static int sample_threads(int rows_bg, int max_seq_len, int sms) {
  return rows_bg > sms && max_seq_len <= 81920 ? 512 : kSampleThreads;
}
// The sample grows with N beyond 2^20 tokens: the bracket's band holds about
// 8 sqrt(k / f) = 8 N / sqrt(S n_s) tokens, so n_s ~ N^2 keeps it within the
// select's shared-memory band capacity.  Rounds of NT * kSampleSlots tokens:
// 1 up to 2^20, ceil((N / 2^20)^2) beyond, at most kSampleMaxRounds (the fast
// path then holds to 2^22 tokens at S = 100; longer rows take the exact slow path).
constexpr int kSampleMaxRounds = 16;
__host__ __device__ __forceinline__ int sample_rounds(int N) {
  if (N <= (1 << 20)) return 1;
  const double x = (double)N / (double)(1 << 20);
  const int r = (int)ceil(x * x);
  return r < kSampleMaxRounds ? r : kSampleMaxRounds;
}
constexpr int kScanNT = 256;               // 8 warps
constexpr int kScanStageTok8 = 1024;       // tokens per ring stage at C = 8 (16 KB)
// Two scan shapes (template NS = ring stages).  NS = 2 with 96-entry candidate
// buffers keeps the CTA at ~53 KB of shared memory and 64 registers: 4 CTAs (32
// warps) per SM, for grids of more than one 3-CTA/SM wave — the scan is latency-
// bound per warp, so occupancy beats ring depth there (cfg3: 3 stages at 3 CTAs/SM
// 59.6 us, 4-5 stages at 2 CTAs/SM 65 us, 2 stages at 4 CTAs/SM 57.9 us).  Smaller
// grids (cfg2, cfg4 turn 0: a partial wave) keep NS = 3 at 3 CTAs/SM, whose deeper
// ring serves a lone CTA better (cfg2 S = 50: 59.4 vs 63.3 us).
__host__ __device__ constexpr int scan_cand_cap(int ns) { return ns == 2 ? 96 : 128; }
__host__ __device__ constexpr int scan_min_blocks(int ns, int g) { return ns == 2 && g < 8 ? 4 : 3; }
constexpr int kSelNT = 256;           // 4 CTAs per SM: B*Hq = 512 rows in one wave
constexpr int kSelCap = 24576;             // band entries cached per row (keys + tokens: 192 KB)
constexpr int kTieCap = 2048;
#ifndef SD_SCAN_HALF
#define SD_SCAN_HALF 2  // half-chunk scan CTAs at the end: (this * SMs) / 2 items (4: 195.3, 2: 194.1, 0: 195.1 us)
#endif
#ifndef SD_SEL_UQ
#define SD_SEL_UQ 6  // select, pair regions: entries per lane requested with the region count
#endif

// The two sample order statistics that bracket the k-th key (k_fused.cu header):
// r_lo = ceil(k f + z sqrt(k f (1-f)) + 1), r_hi = floor(k f - z sqrt(...)),
// f = n_s / N; the whole row sampled: both = k.  fp32 (the bracket is a filter
// the select verifies, so only determinism matters; fp64 here cost ~200
// instructions per thread of the sample kernel).
__device__ __forceinline__ void sample_ranks(int k, int n_s, int N, int* r_lo, int* r_hi) {
  if (n_s >= N) {
    *r_lo = *r_hi = k;
    return;
  }
  const float f = __fdiv_rn((float)n_s, (float)N);
  const float mu = (float)k * f, sd = sqrtf(mu * (1.f - f));
  *r_lo = (int)ceilf(mu + kBracketZ * sd + 1.f);
  *r_hi = (int)floorf(mu - kBracketZ * sd);
}

__device__ __forceinline__ float load_q_elem(const void* q, int q_dtype, size_t e) {
  return q_dtype == SD_F32 ? reinterpret_cast<const float*>(q)[e]
                           : bf_lo(reinterpret_cast<const uint16_t*>(q)[e]);
}

// 2048-bin histograms are stored padded, bin b at hidx(b) = b + b / 64, so
// that a warp reading 64-bin groups (one group per lane) is bank-conflict-free.
constexpr int kHistWords = 2048 + 32;
__device__ __forceinline__ int hidx(uint32_t b) { return (int)(b + (b >> 6)); }

// Warp-level search of a padded 2048-bin histogram (highest bin = largest
// keys) for the bin holding the r-th largest element; returns (bin, residual
// rank).  Two parallel levels: 32 groups of 64 bins, then 32 pairs of bins.
// With `grp` (the 32 group sums, grp[k] = bins [64 k, 64 k + 63]) the first
// level is one load per lane instead of 64.
__device__ __forceinline__ void warp_find_bin(const uint32_t* hist, uint32_t r, int* bin_out, uint32_t* res_out,
                                              const uint32_t* grp = nullptr) {
  const int lane = threadIdx.x & 31;
  const int top = 2047 - 64 * lane;  // lane owns bins [top - 63, top]
  uint32_t sum = 0;
  if (grp) {
    sum = grp[31 - lane];
  } else {
#pragma unroll 16
    for (int i = 0; i < 64; ++i) sum += hist[hidx(top - i)];
  }
  uint32_t incl = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  const uint32_t excl = incl - sum;
  const uint32_t who = __ballot_sync(0xffffffffu, excl < r && incl >= r);
  const int src = who ? __ffs(who) - 1 : 31;
  // level 2: the 64 bins of lane src, two per lane, highest first
  const uint32_t above = __shfl_sync(0xffffffffu, excl, src);
  const int gtop = 2047 - 64 * src;
  const uint32_t c0 = hist[hidx(gtop - 2 * lane)], c1 = hist[hidx(gtop - 2 * lane - 1)];
  const uint32_t pair = c0 + c1;
  uint32_t pin = pair;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, pin, o);
    if (lane >= o) pin += y;
  }
  const uint32_t pex = above + pin - pair;
  const uint32_t who2 = __ballot_sync(0xffffffffu, pex < r && pex + pair >= r);
  const int src2 = who2 ? __ffs(who2) - 1 : 31;
  int bin = gtop - 2 * lane;
  uint32_t res = r - pex;
  if (!(pex + c0 >= r)) {
    bin -= 1;
    res -= c0;
  }
  *bin_out = __shfl_sync(0xffffffffu, bin, src2);
  *res_out = __shfl_sync(0xffffffffu, res, src2);
}

// Group sums of nh padded 2048-bin histograms: grp[h][k] = sum of bins
// [64 k, 64 k + 63] of histogram h (8 threads per group, shuffle reduction).
// All NT threads call it; NT % 32 == 0.
template <int NT>
__device__ __forceinline__ void hist_group_sums(const uint32_t* hist, int nh, uint32_t* grp) {
  for (int base = 0; base < nh * 32 * 8; base += NT) {
    const int i = base + threadIdx.x;  // 8 consecutive threads per group
    const int gi = i >> 3, part = i & 7;
    uint32_t v = 0;
    if (gi < nh * 32) {
      const uint32_t* h = hist + (gi >> 5) * kHistWords;
      const int b0 = (gi & 31) * 64 + part * 8;
#pragma unroll
      for (int k = 0; k < 8; ++k) v += h[hidx(b0 + k)];
    }
    v += __shfl_xor_sync(0xffffffffu, v, 1);
    v += __shfl_xor_sync(0xffffffffu, v, 2);
    v += __shfl_xor_sync(0xffffffffu, v, 4);
    if (part == 0 && gi < nh * 32) grp[gi] = v;
  }
}

// two independent fp32 fma's in one FFMA2 (bit-identical to two fmaf)
__device__ __forceinline__ void ffma2(float& a0, float& a1, float x0, float x1, float y) {
  unsigned long long r;
  const unsigned long long a = ((unsigned long long)__float_as_uint(a1) << 32) | __float_as_uint(a0);
  const unsigned long long xx = ((unsigned long long)__float_as_uint(x1) << 32) | __float_as_uint(x0);
  const unsigned long long yy = ((unsigned long long)__float_as_uint(y) << 32) | __float_as_uint(y);
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(xx), "l"(yy), "l"(a));
  a0 = __uint_as_float((uint32_t)r);
  a1 = __uint_as_float((uint32_t)(r >> 32));
}

// Predicated candidate store (no branch): {x, y} -> shared [a2], code -> shared [at] when p.
__device__ __forceinline__ void st_cand_pred(bool p, uint32_t a2, float x, float y, uint32_t at, uint16_t code) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %0, 0;\n\t"
      "@q st.shared.v2.f32 [%1], {%2, %3};\n\t@q st.shared.u16 [%4], %5;\n}" ::"r"((int)p),
      "r"(a2), "f"(x), "f"(y), "r"(at), "h"(code)
      : "memory");
}

// Float threshold equivalent to key(s) >= lo on finite scores.
__device__ __forceinline__ float thresh_lo(uint32_t lo) {
  if (lo <= 0x007FFFFFu) return -INFINITY;  // below key(-inf): every finite score
  if (lo >= 0xFF800000u) return INFINITY;   // above key(+inf): none
  return key_score(lo);
}

// --------------------------------------------------------------------------- 1. sample
// One CTA per (b, g) for its G q-heads (the sampled sketch rows are loaded once):
// score the deterministic page-strided sample (every spg-th page, <= 4096
// tokens) with the SAME fp32 fma chain as the scan; the scores stay in
// registers.  The r_lo-th / r_hi-th largest sample keys of each head are found
// in two histogram passes (11 + 8 key bits): tau_lo = floor of the 19-bit bin
// holding the r_lo-th key, tau_hi = ceiling of the bin holding the r_hi-th
// (a bin is 1/4096 of a binade, so the bracket is set by the sample
// statistics, not by the binning).
constexpr int kSampleBits1 = 11, kSampleBits2 = 8;
constexpr int kSampleSh1 = 32 - kSampleBits1, kSampleSh2 = kSampleSh1 - kSampleBits2;  // 21, 13

// bin of the r-th largest element of a 256-bin histogram (one warp); (bin, residual)
__device__ __forceinline__ void warp_find_bin256(const uint32_t* h, uint32_t r, int* bin_out, uint32_t* res_out) {
  const int lane = threadIdx.x & 31;
  const int top = 255 - 8 * lane;  // lane owns bins [top - 7, top]
  uint32_t c[8], sum = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    c[i] = h[top - i];
    sum += c[i];
  }
  uint32_t incl = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  uint32_t above = incl - sum;
  const uint32_t who = __ballot_sync(0xffffffffu, above < r && incl >= r);
  const int src = who ? __ffs(who) - 1 : 31;
  int bin = top - 7;
  uint32_t res = 1;
  bool found = false;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    if (!found && above + c[i] >= r) {
      bin = top - i;
      res = r - above;
      found = true;
    }
    above += c[i];
  }
  *bin_out = __shfl_sync(0xffffffffu, bin, src);
  *res_out = __shfl_sync(0xffffffffu, res, src);
}

// GG = the GQA group size, G = the heads one CTA handles (GG / G CTAs per (b, g)
// share the group's sample rows when there are few (b, g) rows).
// MULTI: rows longer than 2^20 tokens possible (sample_rounds > 1).
template <int GG, class Sk, int NT, int G, bool MULTI>
__global__ void __launch_bounds__(NT, NT <= 512 ? 2 : 1) sbs_sample_kernel(
    const void* __restrict__ q, int q_dtype, const void* __restrict__ sk, const int* __restrict__ channel_ids,
    int C, const int* __restrict__ page_table, const int* __restrict__ seq_lens, int max_len, int max_pages, int Hkv,
    BudgetDev bud, uint32_t* __restrict__ thr, int* __restrict__ counters) {
  constexpr int CAP = NT * kSampleSlots;
  extern __shared__ __align__(128) unsigned char smem[];
  uint32_t* hist1 = reinterpret_cast<uint32_t*>(smem);  // [G][kHistWords] padded 2048-bin
  uint32_t* hist2 = hist1 + G * kHistWords;              // [G][2][256]
  float* qc = reinterpret_cast<float*>(hist2 + G * 512);  // [G][C]
  unsigned char* s_qrow = reinterpret_cast<unsigned char*>(qc + G * C);  // [G][kD] q dtype (fp32 at most)
  int* s_ch = reinterpret_cast<int*>(s_qrow + (size_t)G * kD * 4);        // [C]
  uint32_t* s_grp = reinterpret_cast<uint32_t*>(s_ch + C);               // [G][32] level-1 group sums
  __shared__ int s_bin1[G][2];
  __shared__ uint32_t s_res[G][2];
  __shared__ uint32_t s_lohi[G][2];
  constexpr int kParts = GG / G;
  // the scan grid may launch now: its CTAs stage their page ids and first
  // sketch stages, then wait (griddepcontrol.wait) for this grid to complete
  pdl_launch_dependents();
  pdl_wait();  // (PDL-launched: the preceding kernel of the stream has finished)
  const int part = blockIdx.x % kParts, bg = blockIdx.x / kParts, b = bg / Hkv, g = bg - b * Hkv;
  const int j0 = part * G;  // this CTA's heads: j0 .. j0 + G - 1 of the group
  const int Hq = Hkv * GG;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // the channel ids and the group's whole q rows are requested first (no
  // dependence), then the sample's sketch rows (N -> page ids -> rows is the
  // longest dependent chain); the histogram clearing and the barrier overlap
  const int qb = q_dtype == SD_F32 ? 4 : 2;
  const int chv = tid < C ? __ldg(channel_ids + (size_t)bg * C + tid) : 0;
  const int nq16 = G * kD * qb / 16;
  const uint4* qsrc = reinterpret_cast<const uint4*>(reinterpret_cast<const char*>(q) + (size_t)(b * Hq + g * GG + j0) * kD * qb);
  const uint4 qv = tid < nq16 ? __ldg(qsrc + tid) : make_uint4(0u, 0u, 0u, 0u);
  const int N = seq_len_dev(seq_lens, b, max_len);  // < 1: an empty row (the select reports it)
  const int* pt = page_table + (size_t)b * max_pages;
  const int npg = (max(N, 1) + 15) >> 4;
  const int rounds = MULTI ? sample_rounds(max(N, 1)) : 1;
  const int cap_pages = (CAP >> 4) * rounds;
  const int spg = (npg + cap_pages - 1) / cap_pages;  // page stride
  const int ns_pages = (npg + spg - 1) / spg;
  const int n_slots = ns_pages * 16;
  typename Sk::Raw raw[kSampleSlots];
  int tt[kSampleSlots];
  // sample slot i = tid + NT u + CAP r of round r: token (i / 16) spg 16 + i % 16
  auto load_round = [&](int r) {
#pragma unroll
    for (int u = 0; u < kSampleSlots; ++u) {
      const int i = tid + u * NT + r * CAP;
      const int t = (i >> 4) * spg * 16 + (i & 15);
      tt[u] = (i < n_slots && t < N) ? t : -1;
      if (tt[u] >= 0) raw[u] = Sk::load8(sk, sketch_row_elem(__ldg(pt + (t >> 4)), t & 15, g, Hkv, C));
    }
  };
  load_round(0);
  for (int i = tid; i < G * kHistWords; i += NT) hist1[i] = 0;
  for (int i = tid; i < G * 512; i += NT) hist2[i] = 0;
  if (tid < C) s_ch[tid] = chv;
  if (tid < nq16) reinterpret_cast<uint4*>(s_qrow)[tid] = qv;
  if (tid == 0) {
    if (part == 0) counters[bg] = 0;  // re-arm the gather-attend merge counter of (b, g)
    if (blockIdx.x == 0) counters[gridDim.x / kParts] = 0;  // and the work counter
  }
  __syncthreads();
  for (int i = tid; i < G * C; i += NT) {  // qc[j][c] = q[b][g G + j][channel_ids[b][g][c]]
    const int j = i / C, e = j * kD + s_ch[i - j * C];
    qc[i] = qb == 4 ? reinterpret_cast<const float*>(s_qrow)[e] : bf_lo(reinterpret_cast<const uint16_t*>(s_qrow)[e]);
  }
  __syncthreads();
  if (N < 1) return;
  const RowBudget rbud = row_budget(N, bud);  // NEXT-1: sinks / locals score +inf
  const int k = bud.kfrom ? max(0, shard_row_k(bud, b, N)) : min(rbud.k, N);
  uint32_t key[kSampleSlots][G];
  auto score_round = [&]() {
#pragma unroll
    for (int u = 0; u < kSampleSlots; ++u) {
      float acc[G];
#pragma unroll
      for (int j = 0; j < G; ++j) acc[j] = 0.f;
      if (tt[u] >= 0) {
        sketch_fma8<G, Sk>(raw[u], qc, C, acc);
        if (C > 8) {
          const int t = tt[u];
          const size_t re = sketch_row_elem(__ldg(pt + (t >> 4)), t & 15, g, Hkv, C);
          for (int c0 = 8; c0 < C; c0 += 8) sketch_fma8<G, Sk>(Sk::load8(sk, re + c0), qc + c0, C, acc);
        }
        if (tt[u] < rbud.lo || tt[u] >= rbud.hi) {
#pragma unroll
          for (int j = 0; j < G; ++j) acc[j] = INFINITY;
        }
      }
#pragma unroll
      for (int j = 0; j < G; ++j) key[u][j] = score_key(acc[j]);
    }
  };
  for (int r = 0; r < (MULTI ? rounds : 1); ++r) {
    if (r) load_round(r);
    score_round();
#pragma unroll
    for (int u = 0; u < kSampleSlots; ++u)
#pragma unroll
      for (int j = 0; j < G; ++j)
        if (tt[u] >= 0) atomicAdd(&hist1[j * kHistWords + hidx(key[u][j] >> kSampleSh1)], 1u);
  }
  const int last_sampled = (ns_pages - 1) * spg;
  const int n_s = n_slots - ((last_sampled == npg - 1) ? (npg * 16 - N) : 0);
  int r_lo, r_hi;
  sample_ranks(k, n_s, N, &r_lo, &r_hi);
  const uint32_t ra = (uint32_t)min(r_lo, n_s), rb = (uint32_t)max(r_hi, 1);
  __syncthreads();
  hist_group_sums<NT>(hist1, G, s_grp);
  __syncthreads();
  // level 1: warp 2 j + e finds the 11-bit bin of rank (ra, rb)[e] for head j
  if (warp < 2 * G) {
    const int j = warp >> 1, e = warp & 1;
    int bin;
    uint32_t res;
    warp_find_bin(hist1 + j * kHistWords, e ? rb : ra, &bin, &res, s_grp + j * 32);
    if (lane == 0) {
      s_bin1[j][e] = bin;
      s_res[j][e] = res;
    }
  }
  __syncthreads();
  // level 2: the next 8 key bits inside the two bins of each head
  int bin_lo[G], bin_hi[G];
#pragma unroll
  for (int j = 0; j < G; ++j) {
    bin_lo[j] = s_bin1[j][0];
    bin_hi[j] = s_bin1[j][1];
  }
  for (int r = 0; r < (MULTI ? rounds : 1); ++r) {
    if (MULTI && rounds > 1) {  // one round: the keys are still in registers
      load_round(r);
      score_round();
    }
#pragma unroll
    for (int u = 0; u < kSampleSlots; ++u) {
#pragma unroll
      for (int j = 0; j < G; ++j) {
        const int b1 = (int)(key[u][j] >> kSampleSh1);
        const uint32_t b2 = (key[u][j] >> kSampleSh2) & 255u;
        const bool m0 = tt[u] >= 0 && b1 == bin_lo[j], m1 = tt[u] >= 0 && b1 == bin_hi[j];
        if (__any_sync(0xffffffffu, m0 || m1)) {  // only warps holding a key of a selected bin
          if (m0) atomicAdd(&hist2[(j * 2 + 0) * 256 + b2], 1u);
          if (m1) atomicAdd(&hist2[(j * 2 + 1) * 256 + b2], 1u);
        }
      }
    }
  }
  __syncthreads();
  if (warp < 2 * G) {
    const int j = warp >> 1, e = warp & 1;
    int bin;
    uint32_t res;
    warp_find_bin256(hist2 + (j * 2 + e) * 256, s_res[j][e], &bin, &res);
    if (lane == 0) {
      const uint32_t pre = ((uint32_t)s_bin1[j][e] << kSampleSh1) | ((uint32_t)bin << kSampleSh2);
      s_lohi[j][e] = e ? (pre | ((1u << kSampleSh2) - 1u)) : pre;  // hi: bin ceiling, lo: bin floor
    }
  }
  __syncthreads();
  if (tid < G) {
    uint32_t lo = s_lohi[tid][0], hi = s_lohi[tid][1];
    if (r_lo > n_s) lo = 0u;         // not enough sample mass: every token is a candidate
    if (r_hi < 1) hi = 0xFFFFFFFFu;  // no token is sure
    const size_t row = (size_t)b * Hq + g * GG + j0 + tid;
    // keys for the select; the equivalent float thresholds for the scan
    // (score >= flo <=> key >= lo;  score >= fsure <=> key > hi)
    const float flo = thresh_lo(lo), fsure = hi == 0xFFFFFFFFu ? INFINITY : thresh_lo(hi + 1u);
    reinterpret_cast<uint4*>(thr)[row] = make_uint4(lo, hi, __float_as_uint(flo), __float_as_uint(fsure));
  }
}

// Tensor-core variant for G = 4 q-heads per KV head, C = 8, bf16 sketch (the
// scan's scoring, sd_score.cuh): a warp scores 32 sample tokens (two sampled
// pages) for all 4 heads with one mma.sync, so the sample's scores are the
// scan's bits.  H = heads this CTA brackets (4, or 2 when two CTAs share a
// (b, g)).  Only keys >= 0 (positive scores) enter the level-1 histogram when
// the highest rank needed is within the top quarter of the sample (keys below
// cannot hold it; otherwise every key counts).  Same bracket statistics as
// sbs_sample_kernel.
template <int NT, int H, bool MULTI>
__global__ void __launch_bounds__(NT, NT <= 512 ? 2 : 1) sbs_sample_mma_kernel(
    const void* __restrict__ q, int q_dtype, const uint16_t* __restrict__ sk, const int* __restrict__ channel_ids,
    const int* __restrict__ page_table, const int* __restrict__ seq_lens, int max_len, int max_pages, int Hkv,
    BudgetDev bud, uint32_t* __restrict__ thr, int* __restrict__ counters) {
  constexpr int GG = 4, C = 8;
  constexpr int NWp = NT / 32;
  constexpr int BPR = NWp * kSampleSlots;  // 32-token blocks per round
  constexpr int CAP = BPR * 32;            // sample tokens per round (= NT * kSampleSlots)
  extern __shared__ __align__(128) unsigned char smem[];
  uint32_t* hist1 = reinterpret_cast<uint32_t*>(smem);  // [H][kHistWords] padded 2048-bin
  uint32_t* hist2 = hist1 + H * kHistWords;              // [H][2][256]
  unsigned char* s_qrow = reinterpret_cast<unsigned char*>(hist2 + H * 512);  // [4][kD] q dtype
  int* s_ch = reinterpret_cast<int*>(s_qrow + (size_t)GG * kD * 4);          // [C]
  uint32_t* s_grp = reinterpret_cast<uint32_t*>(s_ch + C);                   // [H][32] level-1 group sums
  __shared__ int s_bin1[H][2];
  __shared__ uint32_t s_res[H][2];
  __shared__ uint32_t s_lohi[H][2];
  constexpr int kParts = GG / H;
  pdl_launch_dependents();  // the scan may launch now (it waits for this grid before reading the bracket)
  pdl_wait();  // (PDL-launched: the preceding kernel of the stream, e.g. the one producing q, has finished)
  const int part = blockIdx.x % kParts, bg = blockIdx.x / kParts, b = bg / Hkv, g = bg - b * Hkv;
  const int j0 = part * H;
  const int Hq = Hkv * GG;
  const int row0 = b * Hq + g * GG;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int qb = q_dtype == SD_F32 ? 4 : 2;
  const int chv = tid < C ? __ldg(channel_ids + (size_t)bg * C + tid) : 0;
  const int nq16 = GG * kD * qb / 16;
  const uint4* qsrc = reinterpret_cast<const uint4*>(reinterpret_cast<const char*>(q) + (size_t)row0 * kD * qb);
  const uint4 qv = tid < nq16 ? __ldg(qsrc + tid) : make_uint4(0u, 0u, 0u, 0u);
  const int N = seq_len_dev(seq_lens, b, max_len);  // < 1: an empty row (the select reports it)
  const int* pt = page_table + (size_t)b * max_pages;
  const int npg = (max(N, 1) + 15) >> 4;
  const int rounds = MULTI ? sample_rounds(max(N, 1)) : 1;
  const int cap_pages = (CAP >> 4) * rounds;
  const int spg = (npg + cap_pages - 1) / cap_pages;  // page stride
  const int ns_pages = (npg + spg - 1) / spg;
  // lane (r, uu) of the MMA: A rows r, r + 8 (page 2 bi) and r, r + 8 (page 2 bi + 1), channels 2 uu, 2 uu + 1;
  // D: tokens tA = r + 16 (uu >> 1), tA + 8 of the block, heads 2 (uu & 1), 2 (uu & 1) + 1
  const int r = lane >> 2, uu = lane & 3;
  uint32_t a[kSampleSlots][4];
  int tA[kSampleSlots];  // absolute token of D rows r (+16) of block slot u; -1: block not sampled
  auto load_round = [&](int rr) {
    int pg[kSampleSlots][2];
#pragma unroll
    for (int u = 0; u < kSampleSlots; ++u) {
      const int bi = warp + NWp * u + BPR * rr;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int sp = 2 * bi + e;
        pg[u][e] = sp < ns_pages ? __ldg(pt + sp * spg) : -1;
      }
    }
#pragma unroll
    for (int u = 0; u < kSampleSlots; ++u) {
      const int bi = warp + NWp * u + BPR * rr;
      tA[u] = 2 * bi < ns_pages ? (2 * bi + (uu >> 1)) * spg * 16 + r : -1;
#pragma unroll
      for (int mm = 0; mm < 4; ++mm) {
        const int e = mm >> 1, slot = 8 * (mm & 1) + r;
        const int t = (2 * bi + e) * spg * 16 + slot;
        a[u][mm] = (pg[u][e] >= 0 && t < N)
                       ? __ldg(reinterpret_cast<const uint32_t*>(sk + sketch_row_elem(pg[u][e], slot, g, Hkv, C)) + uu)
                       : 0u;
      }
    }
  };
  load_round(0);
  for (int i = tid; i < H * kHistWords; i += NT) hist1[i] = 0;
  for (int i = tid; i < H * 512; i += NT) hist2[i] = 0;
  if (tid < C) s_ch[tid] = chv;
  if (tid < nq16) reinterpret_cast<uint4*>(s_qrow)[tid] = qv;
  if (tid == 0) {
    if (part == 0) counters[bg] = 0;  // re-arm the gather-attend merge counter of (b, g)
    if (blockIdx.x == 0) counters[gridDim.x / kParts] = 0;  // and the work counter
  }
  __syncthreads();
  if (N < 1) return;
  const SkMmaQ qm = sk_mma_q(
      [&](int j, int c) {
        const int e = j * kD + s_ch[c];
        return qb == 4 ? reinterpret_cast<const float*>(s_qrow)[e] : bf_lo(reinterpret_cast<const uint16_t*>(s_qrow)[e]);
      },
      q_dtype == SD_F32 ? 3 : 1);
  const RowBudget rbud = row_budget(N, bud);  // NEXT-1: sinks / locals score +inf
  const int k = bud.kfrom ? max(0, shard_row_k(bud, b, N)) : min(rbud.k, N);
  const int last_sampled = (ns_pages - 1) * spg;
  const int n_s = ns_pages * 16 - ((last_sampled == npg - 1) ? (npg * 16 - N) : 0);
  int r_lo, r_hi;
  sample_ranks(k, n_s, N, &r_lo, &r_hi);
  const uint32_t ra = (uint32_t)min(r_lo, n_s), rb = (uint32_t)max(r_hi, 1);
  const uint32_t kmin = 4u * ra <= (uint32_t)n_s ? 0x80000000u : 0u;  // level-1 key floor
  const int hsel = 2 * (uu & 1) - j0;  // this lane's first head, relative to the CTA's
  const bool mine = hsel >= 0 && hsel < H;
  uint32_t key[kSampleSlots][4];  // [u][(token tA | tA + 8) * 2 + head]
  auto score_round = [&]() {
#pragma unroll
    for (int u = 0; u < kSampleSlots; ++u) {
      float d[4];
      sk_mma_score(a[u], qm, d);
#pragma unroll
      for (int x = 0; x < 4; ++x) {
        const int t = tA[u] + 8 * (x >> 1);
        if (t >= 0 && (t < rbud.lo || t >= rbud.hi)) d[x] = INFINITY;
        key[u][x] = (tA[u] >= 0 && t < N) ? score_key(d[x]) : 0u;  // 0: not a sample token
      }
    }
  };
  for (int rr = 0; rr < (MULTI ? rounds : 1); ++rr) {
    if (rr) load_round(rr);
    score_round();
    // branch-free: a key that does not count goes to this lane's pad word of
    // histogram 0 (pad words are never read, hidx skips them)
    uint32_t* const dummy1 = hist1 + 65 * (lane + 1) - 1;
#pragma unroll
    for (int u = 0; u < kSampleSlots; ++u)
#pragma unroll
      for (int x = 0; x < 4; ++x) {
        const uint32_t kk = key[u][x];
        const bool ok = mine && kk >= kmin && kk != 0u;
        atomicAdd(ok ? hist1 + (hsel + (x & 1)) * kHistWords + hidx(kk >> kSampleSh1) : dummy1, 1u);
      }
  }
  __syncthreads();
  hist_group_sums<NT>(hist1, H, s_grp);
  __syncthreads();
  if (warp < 2 * H) {
    const int j = warp >> 1, e = warp & 1;
    int bin;
    uint32_t res;
    warp_find_bin(hist1 + j * kHistWords, e ? rb : ra, &bin, &res, s_grp + j * 32);
    if (lane == 0) {
      s_bin1[j][e] = bin;
      s_res[j][e] = res;
    }
  }
  __syncthreads();
  // level 2: the next 8 key bits inside the two bins of each head
  int bl0 = 0, bh0 = 0, bl1 = 0, bh1 = 0;
  if (mine) {
    bl0 = s_bin1[hsel][0];
    bh0 = s_bin1[hsel][1];
    bl1 = s_bin1[hsel + 1][0];
    bh1 = s_bin1[hsel + 1][1];
  }
  for (int rr = 0; rr < (MULTI ? rounds : 1); ++rr) {
    if (MULTI && rounds > 1) {  // one round: the keys are still in registers
      load_round(rr);
      score_round();
    }
    // only warps holding a key of a selected bin issue (warp-uniform test), to
    // the lane's dummy word when its own key is not one
    uint32_t* const dummy2 = s_grp + H * 32 + lane;
#pragma unroll
    for (int u = 0; u < kSampleSlots; ++u)
#pragma unroll
      for (int x = 0; x < 4; ++x) {
        const uint32_t kk = key[u][x];
        const int j = hsel + (x & 1);
        const int b1 = (int)(kk >> kSampleSh1);
        const uint32_t b2 = (kk >> kSampleSh2) & 255u;
        const bool v = mine && kk != 0u;
        const bool m0 = v && b1 == ((x & 1) ? bl1 : bl0), m1 = v && b1 == ((x & 1) ? bh1 : bh0);
        if (__any_sync(0xffffffffu, m0 || m1)) {
          atomicAdd(m0 ? hist2 + (j * 2 + 0) * 256 + b2 : dummy2, 1u);
          atomicAdd(m1 ? hist2 + (j * 2 + 1) * 256 + b2 : dummy2, 1u);
        }
      }
  }
  __syncthreads();
  if (warp < 2 * H) {
    const int j = warp >> 1, e = warp & 1;
    int bin;
    uint32_t res;
    warp_find_bin256(hist2 + (j * 2 + e) * 256, s_res[j][e], &bin, &res);
    if (lane == 0) {
      const uint32_t pre = ((uint32_t)s_bin1[j][e] << kSampleSh1) | ((uint32_t)bin << kSampleSh2);
      s_lohi[j][e] = e ? (pre | ((1u << kSampleSh2) - 1u)) : pre;  // hi: bin ceiling, lo: bin floor
    }
  }
  __syncthreads();
  if (tid < H) {
    uint32_t lo = s_lohi[tid][0], hi = s_lohi[tid][1];
    if (r_lo > n_s) lo = 0u;         // not enough sample mass: every token is a candidate
    if (r_hi < 1) hi = 0xFFFFFFFFu;  // no token is sure
    const size_t row = (size_t)row0 + j0 + tid;
    const float flo = thresh_lo(lo), fsure = hi == 0xFFFFFFFFu ? INFINITY : thresh_lo(hi + 1u);
    reinterpret_cast<uint4*>(thr)[row] = make_uint4(lo, hi, __float_as_uint(flo), __float_as_uint(fsure));
  }
}

// --------------------------------------------------------------------------- select core (kernel 3.)
// Arguments of the select step (the kernel parameter of sbs_select_kernel).
struct SelArgs {
  const void* q;
  int q_dtype;
  const void* sk;
  const int* channel_ids;
  int C;
  const int* page_table;
  const int* seq_lens;
  int max_len, max_pages, Hkv;
  BudgetDev bud;
  const uint32_t* thr;
  const uint32_t* ent_tok;
  const float* ent_sc;
  const int* ent_cnt;
  int nch;
  uint32_t* fbm;
  int ldw;
  float* scratch;
  int ld;
  int* counts_out;
  int force_fallback;
  int* err;
  int sel_cap;
  int nreg_cap;  // band regions the shared-memory count table holds (more: exact slow path)
};

// the slow path's radix state and the fast path's band histograms share storage
template <int NT, int HPC>
union SelShared {
  SelectSmem<NT> sel;
  uint32_t hist2[HPC][kHistWords];
};

// Dynamic shared memory of select_core: keys, tokens [HPC][sel_cap], ties
// [HPC][kTieCap], q channels [HPC][C], region counts [nreg_cap].
__host__ __device__ constexpr size_t sel_core_smem(int hpc, int sel_cap, int C, int nreg_cap) {
  return (((size_t)4 * hpc * (2 * sel_cap + kTieCap + C) + (size_t)4 * nreg_cap) + 127) & ~(size_t)127;
}

// The select of HPC consecutive q-rows row_base .. (one 256-thread group per
// row); all NT = HPC * 256 threads of the CTA call it.  `smem` = dynamic shared
// memory of at least sel_core_smem(HPC, sel_cap, C, nreg_cap) bytes.
template <int G, class Sk, bool Pair, bool Two>
__device__ __forceinline__ void select_core(const SelArgs& a, int row_base, unsigned char* smem,
                                            SelShared<(Two ? 2 : 1) * kSelNT, Two ? 2 : 1>& ush) {
  const void* __restrict__ q = a.q;
  const int q_dtype = a.q_dtype;
  const void* __restrict__ sk = a.sk;
  const int* __restrict__ channel_ids = a.channel_ids;
  const int C = a.C;
  const int* __restrict__ page_table = a.page_table;
  const int* __restrict__ seq_lens = a.seq_lens;
  const int max_len = a.max_len, max_pages = a.max_pages, Hkv = a.Hkv;
  const BudgetDev bud = a.bud;
  const uint32_t* __restrict__ thr = a.thr;
  const uint32_t* __restrict__ ent_tok = a.ent_tok;
  const float* __restrict__ ent_sc = a.ent_sc;
  const int* __restrict__ ent_cnt = a.ent_cnt;
  const int nch = a.nch;
  uint32_t* __restrict__ fbm = a.fbm;
  const int ldw = a.ldw;
  float* __restrict__ scratch = a.scratch;
  const int ld = a.ld;
  int* __restrict__ counts_out = a.counts_out;
  const int force_fallback = a.force_fallback;
  int* __restrict__ err = a.err;
  const int sel_cap = a.sel_cap;
  // Two (tensor-core scan's head-pair regions, band capacity small enough for
  // 2 CTAs per SM): one CTA per head pair, one 256-thread half per head; the
  // pair's band entries are gathered once for both heads.  Otherwise one CTA
  // per q-head.
  static_assert(!Two || Pair, "two heads per CTA need head-pair regions");
  constexpr int HPC = Two ? 2 : 1;    // heads per CTA
  constexpr int NT = HPC * kSelNT;    // threads per CTA
  constexpr int NW = kScanWarps;
  constexpr int CW = band_region_cap(G);
  uint32_t* keys0 = reinterpret_cast<uint32_t*>(smem);     // [HPC][sel_cap]
  uint32_t* toks0 = keys0 + HPC * sel_cap;                 // [HPC][sel_cap]
  uint32_t* ties0 = toks0 + HPC * sel_cap;                 // [HPC][kTieCap]
  float* qc0 = reinterpret_cast<float*>(ties0 + HPC * kTieCap);  // [HPC][C]
  SelectSmem<NT>& sm = ush.sel;
  __shared__ int s_fb[HPC], s_sure[HPC], s_ntie[HPC], s_n[HPC];
  __shared__ uint32_t s_pre[HPC], s_need[HPC];
  __shared__ int s_shift[HPC], s_prev[HPC], s_done[HPC];

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int h = tid / kSelNT, ht = tid - h * kSelNT, hw = ht >> 5;  // this thread's head slot / index in it
  const int Hq = Hkv * G;
  const int b = row_base / Hq, g = (row_base - b * Hq) / G, j0 = row_base - b * Hq - g * G;
  const int bg = b * Hkv + g;
  const int N = seq_len_dev(seq_lens, b, max_len);  // -1 / 0: SD_DEVERR_SEQLEN below
  const int* pt = page_table + (size_t)b * max_pages;
  for (int i = tid; i < HPC * C; i += NT) {  // (the q channels are used by the slow path only)
    const int hh = i / C, c = i - hh * C;
    const int ch = __ldg(channel_ids + ((size_t)b * Hkv + g) * C + c);
    qc0[i] = load_q_elem(q, q_dtype, (size_t)(row_base + hh) * kD + ch);
  }
  if (tid < HPC) {
    s_fb[tid] = force_fallback;
    s_sure[tid] = 0;
    s_n[tid] = 0;
  }
  pdl_wait();
  const RowBudget rb = row_budget(max(N, 0), bud);
  const int k = bud.kfrom ? (N >= 0 ? shard_row_k(bud, b, N) : -1) : (N >= 1 ? rb.k : 0);
  if (bud.kfrom && N == 0 && k == 0) {  // an empty shard of a valid sequence: no candidates
    if (counts_out && tid < HPC) counts_out[row_base + tid] = 0;
    return;
  }
  if (N < 1 || k > N || (k < 1 && !budget_regions(bud))) {
    if (tid < HPC) {
      set_error(err, SD_DEVERR_SEQLEN);
      if (counts_out) counts_out[row_base + tid] = 0;
    }
    return;
  }
  const int row = row_base + h;  // this half's row
  uint32_t* fr = fbm + (size_t)row * ldw;
  const uint32_t lo = thr[row * 4 + 0], hi = thr[row * 4 + 1];
  const int nw = (N + 31) >> 5;
  __syncthreads();
  const uint32_t lt = (1u << lane) - 1u;
  constexpr int nh = Pair ? 2 : G;
  const int sub = Pair ? (j0 >> 1) : 0, e0 = Pair ? (j0 & 1) : j0;  // score index of head slot 0 (Two: 0)
  // Keep KQ loaded entries (token | mask << 24, HPC scores each) for every head
  // slot whose mask bit they carry: per slot one warp ballot per entry, one
  // shared-memory atomic per warp for the positions.
  auto keep_entries = [&](auto kq_tag, const uint32_t* tk, const float* sc) {
    constexpr int KQ = decltype(kq_tag)::value;
#pragma unroll
    for (int hh = 0; hh < HPC; ++hh) {
      const uint32_t jbit = 1u << (24 + e0 + hh);
      uint32_t* keys = keys0 + hh * sel_cap;
      uint32_t* toks = toks0 + hh * sel_cap;
      uint32_t bal[KQ];
      int tot = 0;
#pragma unroll
      for (int u = 0; u < KQ; ++u) {
        bal[u] = __ballot_sync(0xffffffffu, (tk[u] & jbit) != 0u);
        tot += __popc(bal[u]);
      }
      if (tot) {
        int base = 0;
        if (lane == 0) base = atomicAdd(&s_n[hh], tot);
        base = __shfl_sync(0xffffffffu, base, 0);
#pragma unroll
        for (int u = 0; u < KQ; ++u) {
          const int p = base + __popc(bal[u] & lt);
          if ((bal[u] >> lane) & 1u && p < sel_cap) {
            keys[p] = score_key(sc[u * HPC + hh]);
            toks[p] = tk[u] & 0x00FFFFFFu;
          }
          base += __popc(bal[u]);
        }
      }
    }
  };
  auto sure_count = [&]() {  // the scan's bits of the half's row (all its loads in one round)
    int sure = 0;
    const uint2* fr2 = reinterpret_cast<const uint2*>(fr);  // ldw is even: 8-B aligned rows
    const int nw2 = (nw + 1) >> 1;
#pragma unroll 8
    for (int w = ht; w < nw2; w += kSelNT) {
      uint2 v = fr2[w];
      if (2 * w + 1 >= nw) v.y = 0u;  // the word past N_b is not the scan's
      sure += __popc(v.x) + __popc(v.y);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sure += __shfl_xor_sync(0xffffffffu, sure, o);
    if (lane == 0 && sure) atomicAdd(&s_sure[h], sure);
  };
  if constexpr (Pair) {
    // ---- band entries of the tensor-core scan: one region per (8192-token
    // chunk, head pair), written by the scan CTA's 8 warps (capacity
    // kScanWarps * CW).  Warp w takes chunks w, w + NT/32, ...; its lanes request
    // entries lane + 32 u (u < kUQ) together with the region's count, so the
    // counts, the entries and the sure-count words arrive in one memory round
    // trip; entries past the count are dropped, longer regions finish in rounds
    // of kUT * 32.
    constexpr int kCWC = NW * CW, kSub = kCWC / 2;  // chunk region, its two sub-regions
    constexpr int kUQ = SD_SEL_UQ, kUT = 4;
    const int nchr = (N + kRangeTok - 1) / kRangeTok;
    // kUT-entry-per-lane rounds over entries [i0, cnt) of a sub-region
    auto keep_rest = [&](const uint32_t* rtok, const float* rsc, int i0, int cnt) {
      for (; i0 < cnt; i0 += 32 * kUT) {
        uint32_t tk1[kUT];
        float sc1[kUT * HPC];
#pragma unroll
        for (int u = 0; u < kUT; ++u) {
          const int i = i0 + lane + 32 * u;
          tk1[u] = i < cnt ? rtok[i] : 0u;
#pragma unroll
          for (int hh = 0; hh < HPC; ++hh) sc1[u * HPC + hh] = i < cnt ? rsc[(size_t)i * 2 + hh] : 0.f;
        }
        keep_entries(std::integral_constant<int, kUT>{}, tk1, sc1);
      }
    };
    for (int c0 = warp; c0 < nchr; c0 += NT / 32) {
      const size_t cr = ((size_t)bg * nch + c0) * 2 + sub;
      const uint32_t* rtok = ent_tok + cr * kCWC;
      const float* rsc = ent_sc + cr * kCWC * 2 + e0;
      uint32_t tk[kUQ];
      float sc[kUQ * HPC];
#pragma unroll
      for (int u = 0; u < kUQ; ++u) {
        const int i = lane + 32 * u;
        tk[u] = rtok[i];
        if constexpr (HPC == 2) {
          const float2 v = *reinterpret_cast<const float2*>(rsc + (size_t)i * 2);
          sc[2 * u] = v.x;
          sc[2 * u + 1] = v.y;
        } else {
          sc[u] = rsc[(size_t)i * 2];
        }
      }
      int cnt = ent_cnt[cr * 2], cnt1 = ent_cnt[cr * 2 + 1];  // sub-region 1: a second half-chunk CTA
      if (c0 == warp) sure_count();  // (first pass only) its loads overlap the entries'
      if (cnt > kSub || cnt1 > kSub) {  // region overflow: exact slow path
        for (int hh = 0; hh < HPC; ++hh) s_fb[hh] = 1;
        cnt = cnt1 = 0;
      }
#pragma unroll
      for (int u = 0; u < kUQ; ++u)
        if (lane + 32 * u >= cnt) tk[u] = 0u;
      keep_entries(std::integral_constant<int, kUQ>{}, tk, sc);
      keep_rest(rtok, rsc, 32 * kUQ, cnt);
      keep_rest(rtok + kSub, rsc + (size_t)kSub * 2, 0, cnt1);
    }
    if (warp >= nchr) sure_count();
  } else {
    sure_count();
    // ---- band entries (union format: one region per scan warp, G scores per
    // entry): warp per region over the whole CTA
    int nreg = ((N + kRangeTok - 1) / kRangeTok) * NW;
    if (nreg > a.nreg_cap) {  // count table too small (beyond the shared memory): exact slow path
      nreg = 0;
      if (tid < HPC) s_fb[tid] = 1;
    }
    const size_t reg0 = (size_t)bg * nch * NW;
    auto greg = [&](int r) { return reg0 + r; };
    // region counts -> shared memory in one coalesced pass (overflow: slow path)
    int* s_cnt = reinterpret_cast<int*>(qc0 + HPC * C);  // [nreg]
    for (int r = tid; r < nreg; r += NT) {
      int c = ent_cnt[greg(r)];
      if (c > CW) {
        for (int hh = 0; hh < HPC; ++hh) s_fb[hh] = 1;
        c = 0;
      }
      s_cnt[r] = c;
    }
    __syncthreads();
    // warp per region with RQ regions in flight: entries lane + 32 u (u < UQ) of
    // each are loaded before any is used; longer regions finish in a tail loop.
    constexpr int RQ = 4, UQ = 2;
    for (int rb0 = warp; rb0 < nreg; rb0 += (NT / 32) * RQ) {
      uint32_t tk[RQ * UQ];
      float sc[RQ * UQ * HPC];
      int cnt[RQ];
#pragma unroll
      for (int qq = 0; qq < RQ; ++qq) {
        const int r = rb0 + (NT / 32) * qq;
        cnt[qq] = r < nreg ? s_cnt[r] : 0;
        const uint32_t* rtok = ent_tok + greg(r) * CW;
        const float* rsc = ent_sc + greg(r) * CW * nh + e0;
#pragma unroll
        for (int u = 0; u < UQ; ++u) {
          const int i = lane + 32 * u;
          tk[qq * UQ + u] = i < cnt[qq] ? rtok[i] : 0u;
#pragma unroll
          for (int hh = 0; hh < HPC; ++hh) sc[(qq * UQ + u) * HPC + hh] = i < cnt[qq] ? rsc[(size_t)i * nh + hh] : 0.f;
        }
      }
      keep_entries(std::integral_constant<int, RQ * UQ>{}, tk, sc);
      // tail: regions longer than 32 UQ entries
      for (int qq = 0; qq < RQ; ++qq) {
        const int r = rb0 + (NT / 32) * qq;
        for (int i0 = 32 * UQ; i0 < cnt[qq]; i0 += 32) {
          uint32_t tk1[1] = {0u};
          float sc1[HPC] = {};
          const int i = i0 + lane;
          if (i < cnt[qq]) {
            tk1[0] = ent_tok[greg(r) * CW + i];
#pragma unroll
            for (int hh = 0; hh < HPC; ++hh) sc1[hh] = ent_sc[(greg(r) * CW + i) * nh + e0 + hh];
          }
          keep_entries(std::integral_constant<int, 1>{}, tk1, sc1);
        }
      }
    }
  }
  __syncthreads();
  // ---- per head slot (one 256-thread half each, named barrier 1 + h): the
  // exact r-th largest band key, ties, winners
  auto hsync = [&]() {
    if constexpr (HPC == 1) __syncthreads();
    else asm volatile("bar.sync %0, %1;" ::"r"(1 + h), "r"(kSelNT) : "memory");
  };
  uint32_t* keys = keys0 + h * sel_cap;
  uint32_t* toks = toks0 + h * sel_cap;
  uint32_t* ties = ties0 + h * kTieCap;
  uint32_t* hist2 = ush.hist2[h];
  const int n = s_n[h];
  const int r_need = k - s_sure[h];
  if (ht == 0 && (n > sel_cap || r_need < 0 || r_need > n)) s_fb[h] = 1;
  hsync();
  if (!s_fb[h] && r_need > 0) {
    uint32_t tau;
    int cut = INT_MAX;
    // ---- adaptive radix select of the r-th largest band key (lo <= key <= hi)
    if (ht == 0) {
      const uint32_t span = hi - lo;
      const int bits = span ? 32 - __clz(span) : 1;
      s_prev[h] = bits;
      s_shift[h] = bits > 11 ? bits - 11 : 0;
      s_pre[h] = 0;
      s_need[h] = (uint32_t)r_need;
      s_done[h] = 0;
    }
    hsync();
#pragma unroll 1
    for (int pass = 0; pass < 3 && !s_done[h]; ++pass) {
      for (int i = ht; i < kHistWords; i += kSelNT) hist2[i] = 0;
      hsync();
      const int sh = s_shift[h], prev = s_prev[h];
      const uint32_t pre = s_pre[h], dmask = (1u << (prev - sh)) - 1u;
      for (int i = ht; i < n; i += kSelNT) {
        const uint32_t o = keys[i] - lo;
        if ((uint32_t)((uint64_t)o >> prev) != pre) continue;
        atomicAdd(&hist2[hidx((o >> sh) & dmask)], 1u);
      }
      hsync();
      if (hw == 0) {
        int bin;
        uint32_t res;
        warp_find_bin(hist2, s_need[h], &bin, &res);
        if (lane == 0) {
          s_pre[h] = (uint32_t)(((uint64_t)pre << (prev - sh)) | (uint32_t)bin);
          s_need[h] = res;
          s_prev[h] = sh;
          s_shift[h] = sh > 11 ? sh - 11 : 0;
          s_done[h] = sh == 0;
        }
      }
      hsync();
    }
    tau = lo + s_pre[h];
    const uint32_t need = s_need[h];
    // ---- exact ties at tau: keep the lowest tokens if not all are needed
    if (ht == 0) s_ntie[h] = 0;
    hsync();
    for (int i = ht; i < n; i += kSelNT) {
      if (keys[i] == tau) {
        const int p = atomicAdd(&s_ntie[h], 1);
        if (p < kTieCap) ties[p] = toks[i];
      }
    }
    hsync();
    const int ntie = s_ntie[h];
    if ((uint32_t)ntie > need) {
      if (ntie > kTieCap) {
        if (ht == 0) s_fb[h] = 1;
      } else {
        int cap2 = 1;
        while (cap2 < ntie) cap2 <<= 1;
        for (int i = ntie + ht; i < cap2; i += kSelNT) ties[i] = 0xFFFFFFFFu;
        // ascending bitonic sort of the tied token ids (this half)
        for (int size = 2; size <= cap2; size <<= 1) {
          for (int stride = size >> 1; stride > 0; stride >>= 1) {
            hsync();
            for (int i = ht; i < cap2 / 2; i += kSelNT) {
              const int a = 2 * i - (i & (stride - 1)), c = a + stride;
              const bool up = (a & size) == 0;
              const uint32_t x = ties[a], y = ties[c];
              if ((x > y) == up) {
                ties[a] = y;
                ties[c] = x;
              }
            }
          }
        }
        hsync();
        cut = (int)ties[need - 1];
      }
    }
    hsync();
    if (!s_fb[h]) {
      // ---- band winners into the bitmap
      for (int i = ht; i < n; i += kSelNT) {
        const uint32_t key = keys[i];
        const int t = (int)toks[i];
        if (key > tau || (key == tau && t <= cut)) atomicOr(&fr[t >> 5], 1u << (t & 31));
      }
    }
  }
  __syncthreads();  // the halves join: the slow path uses the whole CTA
  for (int hh = 0; hh < HPC; ++hh) {
    if (!s_fb[hh]) continue;
    // ---- exact slow path for row hh: zero the row, scores -> scratch, radix select, bitmap
    const int rowh = row_base + hh, jh = j0 + hh;
    uint32_t* frh = fbm + (size_t)rowh * ldw;
    const float* qc = qc0 + hh * C;
    if (tid == 0 && err) atomicAdd(err + 1, 1);  // statistics word: fallback rows
    for (int w = tid; w < nw; w += NT) frh[w] = 0u;
    float* sr = scratch + (size_t)rowh * ld;
    if (SkMmaF8<G, Sk>::value && C == 8) {  // the fp8 scan's tensor-core scores, same MMA placement
      const SkMmaF8Q qm8 = sk_mma_q_f8([&](int jj, int c) { return load_q_elem(q, q_dtype, (size_t)(b * Hq + g * G + jj) * kD + __ldg(channel_ids + (size_t)bg * C + c)); });
      const int u = lane & 3, tofs = (lane >> 2) + ((u >> 1) << 4);
      const bool mine = (u & 1) == (jh >> 1);
      for (int t0 = warp * 32; t0 < N; t0 += NT) {
        uint32_t a[4];
        sk_f8_a_global(a, reinterpret_cast<const uint8_t*>(sk), t0, N,
                       [pt, g, Hkv](int t) { return sketch_row_elem(__ldg(pt + (t >> 4)), t & 15, g, Hkv, 8); });
        float d[4];
        sk_mma_score_f8(a, qm8, d);
        const int tA = t0 + tofs, tB = tA + 8;
        const float vA = (jh & 1) ? d[1] : d[0], vB = (jh & 1) ? d[3] : d[2];
        if (mine && tA < N) sr[tA] = (tA < rb.lo || tA >= rb.hi) ? INFINITY : vA;
        if (mine && tB < N) sr[tB] = (tB < rb.lo || tB >= rb.hi) ? INFINITY : vB;
      }
    } else if (SkMma<G, Sk>::value && C == 8) {  // the scan's tensor-core scores, same MMA placement
      const SkMmaQ qm = sk_mma_q([qc, jh](int jj, int c) { return jj == jh ? qc[c] : 0.f; }, q_dtype == SD_F32 ? 3 : 1);
      const int u = lane & 3, tofs = (lane >> 2) + ((u >> 1) << 4);
      const bool mine = (u & 1) == (jh >> 1);
      // 4 blocks per warp in flight (their page ids, then their rows, requested
      // before any is scored: the loop is latency-bound otherwise)
      constexpr int kSU = 4;
      for (int tb = warp * 32; tb < N; tb += kSU * NT) {
        uint32_t a[kSU][4];
#pragma unroll
        for (int x = 0; x < kSU; ++x) {
          const int t0 = tb + x * NT;
          if (t0 < N)
            sk_mma_a_global(a[x], reinterpret_cast<const uint16_t*>(sk), t0, N, [pt, g, Hkv](int t) {
              return sketch_row_elem(__ldg(pt + (t >> 4)), t & 15, g, Hkv, 8);
            });
        }
#pragma unroll
        for (int x = 0; x < kSU; ++x) {
          const int t0 = tb + x * NT;
          if (t0 >= N) break;
          float d[4];
          sk_mma_score(a[x], qm, d);
          const int tA = t0 + tofs, tB = tA + 8;
          const float vA = (jh & 1) ? d[1] : d[0], vB = (jh & 1) ? d[3] : d[2];
          if (mine && tA < N) sr[tA] = (tA < rb.lo || tA >= rb.hi) ? INFINITY : vA;
          if (mine && tB < N) sr[tB] = (tB < rb.lo || tB >= rb.hi) ? INFINITY : vB;
        }
      }
    } else {
      for (int t = tid; t < N; t += NT) {
        const size_t re = sketch_row_elem(__ldg(pt + (t >> 4)), t & 15, g, Hkv, C);
        float acc = 0.f;
        for (int c0 = 0; c0 < C; c0 += 8) sketch_fma8<1, Sk>(Sk::load8(sk, re + c0), qc + c0, C, &acc);
        sr[t] = (t < rb.lo || t >= rb.hi) ? INFINITY : acc;
      }
    }
    __syncthreads();
    auto key_at = [sr](int i) { return score_key(sr[i]); };
    uint32_t ftau, fneed;
    radix_select_block<NT>(key_at, N, (uint32_t)k, sm, &ftau, &fneed);
    emit_block<NT, 4>(key_at, N, ftau, fneed, 0u, sm,
                      [frh](uint32_t, int i, uint32_t) { atomicOr(&frh[i >> 5], 1u << (i & 31)); });
    __syncthreads();
  }
  if (counts_out && tid < HPC) counts_out[row_base + tid] = k;
}

// --------------------------------------------------------------------------- 2. scan
// Every token of (b, g) is classified for each of the G q-heads by the bracket:
//   sure  (key > hi):        its bit is set in the head's selection bitmap fbm
//                            (one ballot word per 32 tokens; every word of the
//                            row below N_b is written, so fbm needs no zeroing);
//   band  (lo <= key <= hi): the token is a union-band entry of the warp's
//                            region (1024 tokens): ent_tok = token | head mask
//                            << 24, ent_sc = the G fp32 scores;
//   below (key < lo):        dropped.
// ent_cnt[b, g, region] = number of entries (> cap: overflow -> slow path).
// C8: sketch width 8 (q channels in registers, one 16-B row per token);
// otherwise a generic C (multiple of 8) with the q channels in shared memory.
template <int G>
__device__ __forceinline__ void store_scores(float* dst, const float (&acc)[G]) {
  if constexpr (G == 1) {
    dst[0] = acc[0];
  } else if constexpr (G == 2) {
    *reinterpret_cast<float2*>(dst) = make_float2(acc[0], acc[1]);
  } else {
#pragma unroll
    for (int j = 0; j < G; j += 4)
      *reinterpret_cast<float4*>(dst + j) = make_float4(acc[j], acc[j + 1], acc[j + 2], acc[j + 3]);
  }
}

template <int G>
__device__ __forceinline__ void load_scores(float (&sc)[G], const float* src) {
  if constexpr (G == 1) {
    sc[0] = src[0];
  } else if constexpr (G == 2) {
    const float2 v = *reinterpret_cast<const float2*>(src);
    sc[0] = v.x;
    sc[1] = v.y;
  } else {
#pragma unroll
    for (int j = 0; j < G; j += 4) {
      const float4 v = *reinterpret_cast<const float4*>(src + j);
      sc[j] = v.x;
      sc[j + 1] = v.y;
      sc[j + 2] = v.z;
      sc[j + 3] = v.w;
    }
  }
}

#ifdef SD_SCAN_TRACE
// debug builds only (-DSD_SCAN_TRACE): per scan CTA {after PDL wait, end} in %globaltimer ns
__device__ unsigned long long g_scan_trace[8192][2];
#endif
template <int G, bool C8, class Sk, int NS>
__global__ void __launch_bounds__(kScanNT, scan_min_blocks(NS, G)) sbs_scan_kernel(
    const void* __restrict__ q, int q_dtype, const char* __restrict__ skb, const int* __restrict__ channel_ids,
    int C, const int* __restrict__ page_table, const int* __restrict__ seq_lens, int max_len, int max_pages, int Hkv,
    const uint32_t* __restrict__ thr, uint32_t* __restrict__ ent_tok, float* __restrict__ ent_sc,
    int* __restrict__ ent_cnt, uint32_t* __restrict__ fbm, int ldw, int nch, BudgetDev bud, int n_half) {
  constexpr int kScanStages = NS;                    // ring stages
  constexpr int kScanCandCap = scan_cand_cap(NS);    // candidate buffer per warp (x2 entries on the MMA path)
  constexpr int NW = kScanNT / 32;
  static_assert(NW == kScanWarps, "one band region per scan warp");
  constexpr int CW = band_region_cap(G);
  constexpr bool kF8 = C8 && SkMmaF8<G, Sk>::value;              // fp8 sketch on the tensor cores
  constexpr bool kMma = C8 && (SkMma<G, Sk>::value || kF8);      // tensor-core scores (sd_score.cuh)
  // stage rows copied by the warp that scores them (bf16 rows; fp8 rows on the tensor-core path)
  constexpr bool kWarpLocal = C8 && (Sk::kBytes == 2 || SkMmaF8<G, Sk>::value);
  constexpr int kWords = kRangeTok / 32;              // bitmap words of the chunk, per head
  // per-warp candidate buffer: (token, head pair) entries on the tensor-core
  // path, (token) entries otherwise; flushed (phase 2) before a block could overflow it
  constexpr int kCap = kMma ? 2 * kScanCandCap : kScanCandCap;
  constexpr int kPerBlk = kMma ? 64 : 32;  // new candidates per warp per 32-token block, at most
  extern __shared__ __align__(128) unsigned char smem[];
  const int rowb = C * Sk::kBytes;                        // one token's sketch row
  const int stage_tok = (kScanStageTok8 * 8 / C) & ~31;  // whole bitmap words per stage
  const int stage_bytes = kScanStageTok8 * 16;            // ring slot size
  unsigned char* ring = smem;
  float* qc = reinterpret_cast<float*>(ring + (size_t)kScanStages * stage_bytes);        // [G][C]
  int* s_pages = reinterpret_cast<int*>(qc + G * C);                                      // [kRangeTok / 16]
  uint32_t* s_words = reinterpret_cast<uint32_t*>(s_pages + kRangeTok / 16);              // [G][kWords]
  float* c_sc_all = reinterpret_cast<float*>(s_words + G * kWords);                       // [NW][kScanCandCap][G]
  uint16_t* c_tok_all = reinterpret_cast<uint16_t*>(c_sc_all + NW * G * kScanCandCap);    // [NW][2 kScanCandCap]

  // 1-D grid in (b, g)-major, chunk-minor order; the last n_half items (the
  // final wave, kMma path only) run as two CTAs of half a chunk each, so the
  // scan's tail is half as long
  const int n_items = (int)gridDim.x - n_half;  // items = B * Hkv * nch
  const int nfull = n_items - n_half;
  int item = blockIdx.x, half = -1;
  if (item >= nfull) {
    half = (item - nfull) & 1;
    item = nfull + ((item - nfull) >> 1);
  }
  const int bg = item / nch, b = bg / Hkv, g = bg - b * Hkv;
  const int Hq = Hkv * G;
  const int row0 = b * Hq + g * G;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int chunk = item - bg * nch;
  const int t0 = chunk * kRangeTok + (half == 1 ? kRangeTok / 2 : 0);
  const int len = half < 0 ? kRangeTok : kRangeTok / 2;  // tokens of this CTA
  const size_t reg = ((size_t)bg * nch + chunk) * NW + warp;
  // kMma: one band region per (chunk, head pair) shared by the CTA's warps
  // (positions from a shared-memory counter per pair), two sub-regions of
  // kSubCap (sub-region 1: the second half-chunk CTA), a count per sub-region
  const size_t creg = (size_t)bg * nch + chunk;
  constexpr int kChunkCap = NW * CW, kSubCap = kChunkCap / 2;
  const int sr = half == 1 ? 1 : 0;
  __shared__ int s_bc[2];
  // ---- prologue: every global input is requested before anything waits on
  // one (N_b, the chunk's page ids, the channel ids, the G q rows, then the
  // brackets once the sample kernel has finished), so the CTA start costs one
  // memory round trip instead of four
  const int qb = q_dtype == SD_F32 ? 4 : 2;
  const int N = max(0, seq_len_dev(seq_lens, b, max_len));  // out of range: an empty row
  const int* pt = page_table + (size_t)b * max_pages + (t0 >> 4);
  const int np_max = min(len / 16, max_pages - (t0 >> 4));  // page ids past N_b are never used
  constexpr int kPgPerThr = kRangeTok / 16 / kScanNT;
  int pgv[kPgPerThr];
#pragma unroll
  for (int u = 0; u < kPgPerThr; ++u) pgv[u] = tid + u * kScanNT < np_max ? __ldg(pt + tid + u * kScanNT) : 0;
  const int chv = tid < C ? __ldg(channel_ids + (size_t)bg * C + tid) : 0;
  const int nq16 = G * kD * qb / 16;  // the group's q rows in 16-B pieces
  const uint4* qsrc = reinterpret_cast<const uint4*>(reinterpret_cast<const char*>(q) + (size_t)row0 * kD * qb);
  uint4 qv[(8 * kD * 4 / 16 + kScanNT - 1) / kScanNT];
#pragma unroll
  for (int u = 0; u < (int)(sizeof(qv) / sizeof(uint4)); ++u)
    if (tid + u * kScanNT < nq16) qv[u] = __ldg(qsrc + tid + u * kScanNT);
  for (int i = tid; i < G * kWords; i += kScanNT) s_words[i] = 0u;
  if (tid < 2) s_bc[tid] = 0;
  // the chunk's first ring stages do not depend on the sample kernel: they are
  // requested before the PDL wait (the sample kernel lets this grid launch at
  // its start), so the scan's first copies overlap the sample
  const int ntok = max(0, min(N - t0, len));
  // the q rows and channel ids are staged in the candidate area (unused until phase 1)
  unsigned char* s_qrow = reinterpret_cast<unsigned char*>(c_sc_all);        // [G][kD] q dtype
  int* s_ch = reinterpret_cast<int*>(s_qrow + (size_t)G * kD * 4);            // [C]
#pragma unroll
  for (int u = 0; u < kPgPerThr; ++u) s_pages[tid + u * kScanNT] = pgv[u];
  if (tid < C) s_ch[tid] = chv;
#pragma unroll
  for (int u = 0; u < (int)(sizeof(qv) / sizeof(uint4)); ++u)
    if (tid + u * kScanNT < nq16) reinterpret_cast<uint4*>(s_qrow)[tid + u * kScanNT] = qv[u];
  __syncthreads();
  auto qf = [&](int j, int c) {  // q[b][g G + j][channel_ids[b][g][c]]
    const int e = j * kD + s_ch[c];
    return qb == 4 ? reinterpret_cast<const float*>(s_qrow)[e] : bf_lo(reinterpret_cast<const uint16_t*>(s_qrow)[e]);
  };
  const int nst = (ntok + stage_tok - 1) / stage_tok;
  const int cpt = rowb >> 4;  // 16-B chunks per token (0 for the 8-B fp8 rows)
  // C8: thread tid copies 16-B chunk tid + 256 u of a stage (kTpc tokens each):
  // page (tid * kTpc >> 4) + 16 kTpc u of the stage, slot (tid * kTpc) & 15
  constexpr int kRowB = 8 * Sk::kBytes;  // C8: one token's sketch row (16 B bf16, 8 B fp8)
  constexpr int kTpc = 16 / kRowB;       // C8: tokens per 16-B copy
  const char* tb = skb + ((size_t)g * kPS + ((tid * kTpc) & 15)) * kRowB;
  // (one opaque 64-bit base: each copy address is then a single IMAD.WIDE.U32)
  asm("mov.b64 %0, %0;" : "+l"(tb));
  const uint32_t page_bytes = (uint32_t)Hkv * kPS * kRowB;
  // stage s into ring slot `slot` (== s % kScanStages, kept by the caller)
  auto issue = [&](int s, int slot) {
    if (s < nst) {
      unsigned char* st = ring + (size_t)slot * stage_bytes;
      if (C8 && SkMmaF8<G, Sk>::value) {
        // fp8 rows, tensor-core path: warp w copies its own 4 blocks of 32 tokens
        // (stage tokens 256 j + 32 w + [0, 32)), 2 tokens per 16-B copy, so a warp
        // only waits for its own lanes' copies
        const bool whole = (s + 1) * kScanStageTok8 <= ntok;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int c = lane + 32 * e, ti = 256 * (c >> 4) + 32 * warp + 2 * (c & 15);
          if (whole || s * kScanStageTok8 + ti < ntok) {
            const int pg = s_pages[(s * kScanStageTok8 + ti) >> 4];
            const char* src = skb + ((size_t)((uint32_t)pg * Hkv + g) * kPS + (ti & 15)) * 8;
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(st + (size_t)ti * 8)), "l"(src)
                         : "memory");
          }
        }
      } else if (C8) {
        const int* sp = s_pages + (s * kScanStageTok8 >> 4) + ((tid * kTpc) >> 4);
        if ((s + 1) * kScanStageTok8 <= ntok) {  // full stage: plain copies
          // every page id is read before the first copy is issued: the copies then
          // issue back to back (no shared-memory load between two LDGSTS)
          constexpr int kU = kScanStageTok8 / kScanNT / kTpc;
          uint32_t pgu[kU];
#pragma unroll
          for (int u = 0; u < kU; ++u) pgu[u] = (uint32_t)sp[u * (kScanNT * kTpc >> 4)];
#pragma unroll
          for (int u = 0; u < kU; ++u) {
            const uint32_t d = smem_u32(st + (size_t)(tid + u * kScanNT) * 16);
            const char* src = tb + (size_t)pgu[u] * page_bytes;
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
          }
        } else {  // the range's tail: only the pages that exist (rows >= N are masked)
#pragma unroll
          for (int u = 0; u < kScanStageTok8 / kScanNT / kTpc; ++u) {
            const int ti = tid + u * kScanNT;  // 16-B chunk: tokens kTpc ti ..
            if (s * kScanStageTok8 + ti * kTpc < ntok) {
              const uint32_t d = smem_u32(st + (size_t)ti * 16);
              const char* src = tb + (size_t)(uint32_t)sp[u * (kScanNT * kTpc >> 4)] * page_bytes;
              asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
            }
          }
        }
      } else {
        const int nq = min(stage_tok, ntok - s * stage_tok) * cpt;
        for (int qd = tid; qd < nq; qd += kScanNT) {
          const int ti = qd / cpt, c = qd - ti * cpt;
          const int i = s * stage_tok + ti;  // chunk-relative token
          const char* src = skb + (sketch_row_elem(s_pages[i >> 4], i & 15, g, Hkv, C) + c * 8) * 2;
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(st + (size_t)qd * 16)), "l"(src)
                       : "memory");
        }
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
#pragma unroll
  for (int s = 0; s < kScanStages - 1; ++s) issue(s, s);
  pdl_wait();  // the bracket comes from the sample kernel
#ifdef SD_SCAN_TRACE
  if (tid == 0) g_scan_trace[blockIdx.y * gridDim.x + blockIdx.x][0] = globaltimer_ns();
#endif
  float2 thv[G];  // {flo, fsure} per head, converted by the sample kernel
  // (written by the PDL primary while this grid may already run: coherent
  // L2 loads, not the read-only path)
#pragma unroll
  for (int j = 0; j < G; ++j) thv[j] = __ldcg(reinterpret_cast<const float2*>(thr) + 2 * (row0 + j) + 1);
  if (ntok == 0) {
    if (kMma) {
      if (tid < 2) ent_cnt[(creg * 2 + tid) * 2 + sr] = 0;
      if (half < 0 && tid < 2) ent_cnt[(creg * 2 + tid) * 2 + 1] = 0;
    } else if (lane == 0) {
      ent_cnt[reg] = 0;
    }
    pdl_launch_dependents();
    return;
  }

  float qr[G][8];
  SkMmaQ qm;
  SkMmaF8Q qm8;
  if constexpr (kF8) {
    qm8 = sk_mma_q_f8(qf);
    qm.np = 8;  // phase-1 selector: the fp8 path
  } else if constexpr (kMma) {
    qm = sk_mma_q(qf, q_dtype == SD_F32 ? 3 : 1);
  } else if (C8) {
#pragma unroll
    for (int j = 0; j < G; ++j)
#pragma unroll
      for (int c = 0; c < 8; ++c) qr[j][c] = qf(j, c);
  } else {
    for (int i = tid; i < G * C; i += kScanNT) qc[i] = qf(i / C, i - (i / C) * C);
  }
  __syncthreads();  // the staged q rows are read; the candidate area is free
  const RowBudget rb = row_budget(N, bud);
  float flo[G], fsure[G];
#pragma unroll
  for (int j = 0; j < G; ++j) {
    flo[j] = thv[j].x;
    fsure[j] = thv[j].y;  // key > hi  <=>  s >= fsure
  }
  const uint32_t lt_mask = (1u << lane) - 1u;
  // band entries and selection words are read by the select right after this
  // kernel: keep them in L2 ahead of the streamed sketch (evict-last stores)
  const uint64_t pol_keep = l2_policy_evict_last();
  uint32_t* rtok = ent_tok + reg * CW;
  float* rsc = ent_sc + reg * CW * G;
  float* c_sc = c_sc_all + warp * G * kScanCandCap;  // this warp's candidates ([p][G])
  uint16_t* c_tok = c_tok_all + warp * kScanCandCap;
  int wn = 0;   // candidates buffered by this warp (chunk-relative tokens)
  int wc = 0;   // band entries written (union format)
  // kMma: this lane's head pair p = u & 1 (phase 1); the thresholds of both pairs (phase 2)
  const int pm_r = lane >> 2, pm_u = lane & 3, pm_p = pm_u & 1;
  const float pm_fla0 = flo[0], pm_fla1 = flo[G > 1 ? 1 : 0], pm_flb0 = flo[G > 2 ? 2 : 0], pm_flb1 = flo[G > 3 ? 3 : 0];
  const float pm_fsa0 = fsure[0], pm_fsa1 = fsure[G > 1 ? 1 : 0], pm_fsb0 = fsure[G > 2 ? 2 : 0],
              pm_fsb1 = fsure[G > 3 ? 3 : 0];
  const float pm_fl0 = pm_p ? pm_flb0 : pm_fla0, pm_fl1 = pm_p ? pm_flb1 : pm_fla1;
  // candidate code of token tA = blk + pm_r + 16 (pm_u >> 1) (< 2^15, no carry into bit 15):
  // (stage-relative block start) + this lane's constant (offset | pair << 15)
  const int pm_lc = (warp * 32 + pm_r + ((pm_u >> 1) << 4)) | (pm_p << 15);
  float2* pm_c2 = reinterpret_cast<float2*>(c_sc_all) + warp * 2 * kScanCandCap;  // [2 * kScanCandCap]
  uint16_t* pm_ct = c_tok_all + warp * 2 * kScanCandCap;
  const uint32_t pm_c2_s = smem_u32(pm_c2), pm_ct_s = smem_u32(pm_ct);  // shared-window addresses

  // ---- phase 2: classify the buffered candidates, one per lane: sure bits into
  // the chunk's words (shared-memory atomics), band tokens into the region
  auto flush = [&]() {
    __syncwarp();
    if constexpr (kMma) {
      for (int c0 = 0; c0 < wn; c0 += 32) {
        const int ci = c0 + lane;
        const bool have = ci < wn;
        const uint32_t code = have ? (uint32_t)pm_ct[ci] : 0u;
        const float2 v = have ? pm_c2[ci] : make_float2(-INFINITY, -INFINITY);
        const int i = (int)(code & 0x7FFFu), p = (int)(code >> 15);
        const bool s0 = v.x >= (p ? pm_fsb0 : pm_fsa0), s1 = v.y >= (p ? pm_fsb1 : pm_fsa1);
        uint32_t* sw = s_words + (2 * p) * kWords + (i >> 5);
        if (s0) atomicOr(sw, 1u << (i & 31));
        if (s1) atomicOr(sw + kWords, 1u << (i & 31));
        const uint32_t m = (!s0 && v.x >= (p ? pm_flb0 : pm_fla0) ? 1u : 0u) |
                           (!s1 && v.y >= (p ? pm_flb1 : pm_fla1) ? 2u : 0u);
        const uint32_t b0 = __ballot_sync(0xffffffffu, m && !p), b1 = __ballot_sync(0xffffffffu, m && p);
        int base = 0;  // lane 0: pair 0's base, lane 1: pair 1's
        if (lane < 2 && (lane ? b1 : b0)) base = atomicAdd(&s_bc[lane], __popc(lane ? b1 : b0));
        const int base0 = __shfl_sync(0xffffffffu, base, 0), base1 = __shfl_sync(0xffffffffu, base, 1);
        if (m) {
          const int pos = (p ? base1 : base0) + __popc((p ? b1 : b0) & lt_mask);
          if (pos < kSubCap) {
            const size_t e = (creg * 2 + p) * kChunkCap + sr * kSubCap + pos;
            st_keep_u32(ent_tok + e, (uint32_t)(t0 + i) | (m << 24), pol_keep);
            st_keep_f2(reinterpret_cast<float2*>(ent_sc) + e, v, pol_keep);
          }
        }
      }
    } else {
      for (int c0 = 0; c0 < wn; c0 += 32) {
        const int ci = c0 + lane;
        const bool have = ci < wn;
        const int i = have ? (int)c_tok[ci] : 0;
        float sc[G];
        uint32_t bm = 0;
        load_scores<G>(sc, c_sc + (have ? ci : 0) * G);
#pragma unroll
        for (int j = 0; j < G; ++j) {
          if (!have) sc[j] = -INFINITY;
          if (sc[j] >= fsure[j]) atomicOr(&s_words[j * kWords + (i >> 5)], 1u << (i & 31));
          else if (sc[j] >= flo[j]) bm |= 1u << j;
        }
        const uint32_t bb = __ballot_sync(0xffffffffu, bm != 0u);
        if (bb) {
          const int pos = wc + __popc(bb & lt_mask);
          if (bm && pos < CW) {
            rtok[pos] = (uint32_t)(t0 + i) | (bm << 24);
            store_scores<G>(rsc + (size_t)pos * G, sc);
          }
          wc += __popc(bb);
        }
      }
    }
    __syncwarp();
    wn = 0;
  };

  const uint32_t ring_s = smem_u32(ring);
  int slot = 0;  // s % kScanStages
  for (int s = 0; s < nst; ++s) {
    const int slot_prev = slot == 0 ? kScanStages - 1 : slot - 1;  // (s + kScanStages - 1) % kScanStages
    issue(s + kScanStages - 1, slot_prev);
    asm volatile("cp.async.wait_group %0;" ::"n"(kScanStages - 1) : "memory");
    // bf16 rows at C = 8: thread tid copies tokens tid + 256 u of a stage, which
    // are exactly the 32-token blocks its warp scores, so a warp only waits for
    // its own lanes' copies (no CTA barrier per stage); otherwise the CTA syncs
    if constexpr (kWarpLocal) __syncwarp();
    else __syncthreads();
    const unsigned char* st = ring + (size_t)slot * stage_bytes;
    const uint32_t st_w = ring_s + (uint32_t)(slot * stage_bytes) + (uint32_t)warp * 32u * 16u;  // this warp's first block
    const int cb = s * stage_tok;                   // chunk-relative first token of the stage
    const int lim = min(stage_tok, ntok - cb);      // valid tokens of this stage
    const int tbase = t0 + cb;                      // first token of the stage
    const bool edge_stage = tbase < rb.lo || tbase + lim > rb.hi;  // touches the sink / local regions
    // ---- phase 1: score every token; keep the candidates (key >= lo for some head)
    if constexpr (kMma) {
      // one MMA per 32-token block (sd_score.cuh): lane (r, u) holds heads 2p,
      // 2p+1 (p = u & 1) of tokens tA, tA + 8; each (token, pair) with a score
      // >= lo becomes a candidate: its 2 scores and token | p << 15.  NP = the
      // q parts of sk_mma_q (1: bf16 q); FULL = a whole stage with no sink /
      // local tokens (no per-token range checks).
      auto phase1 = [&](auto np_tag, auto full_tag) {
        constexpr int NP = decltype(np_tag)::value;
        constexpr bool FULL = decltype(full_tag)::value;
        // two 32-token blocks per flush check: both fragments and MMAs are
        // issued before either block's compares (no control dependence between them)
        constexpr int kB = 2;
#pragma unroll 2
        for (int i0 = 0; i0 < kScanStageTok8; i0 += kB * kScanNT) {
          if (wn > kCap - kB * kPerBlk) flush();
          float d[kB][4];
#pragma unroll
          for (int h = 0; h < kB; ++h) {
            uint32_t a[4];
            if constexpr (NP == 8) {  // fp8 rows of 8 B: the scores of sk_mma_score_f8
              sk_f8_a_smem(a, smem_u32(st) + (uint32_t)(i0 + h * kScanNT + warp * 32) * 8u);
              sk_mma_score_f8(a, qm8, d[h]);
            } else {
              sk_mma_a_smem(a, st_w + (uint32_t)(i0 + h * kScanNT) * 16u);
              d[h][0] = d[h][1] = d[h][2] = d[h][3] = 0.f;
              sk_mma(d[h], a, qm.b[0]);  // the accumulation order of sk_mma_score
              if constexpr (NP > 1) {
                sk_mma(d[h], a, qm.b[1]);
                sk_mma(d[h], a, qm.b[2]);
              }
            }
          }
#pragma unroll
          for (int h = 0; h < kB; ++h) {
            const int blk = i0 + h * kScanNT + warp * 32;
            const int tA = blk + pm_r + ((pm_u >> 1) << 4), tB = tA + 8;
            if constexpr (!FULL) {
              if (edge_stage) {  // NEXT-1: sink / local tokens rank above every score
                if (tbase + tA < rb.lo || tbase + tA >= rb.hi) d[h][0] = d[h][1] = INFINITY;
                if (tbase + tB < rb.lo || tbase + tB >= rb.hi) d[h][2] = d[h][3] = INFINITY;
              }
            }
            bool cA = d[h][0] >= pm_fl0 || d[h][1] >= pm_fl1;
            bool cB = d[h][2] >= pm_fl0 || d[h][3] >= pm_fl1;
            if constexpr (!FULL) {
              cA = cA && tA < lim;
              cB = cB && tB < lim;
            }
            const uint32_t bA = __ballot_sync(0xffffffffu, cA), bB = __ballot_sync(0xffffffffu, cB);
            const int nA = __popc(bA);
            const int pA = wn + __popc(bA & lt_mask), pB = wn + nA + __popc(bB & lt_mask);
            const int code0 = cb + i0 + h * kScanNT + pm_lc;  // == (cb + tA) | pm_p << 15
            st_cand_pred(cA, pm_c2_s + 8u * (uint32_t)pA, d[h][0], d[h][1], pm_ct_s + 2u * (uint32_t)pA,
                         (uint16_t)code0);
            st_cand_pred(cB, pm_c2_s + 8u * (uint32_t)pB, d[h][2], d[h][3], pm_ct_s + 2u * (uint32_t)pB,
                         (uint16_t)(code0 + 8));
            wn += nA + __popc(bB);
          }
        }
      };
      const bool full = lim == kScanStageTok8 && !edge_stage;
      if constexpr (kF8) {
        if (full) phase1(std::integral_constant<int, 8>{}, std::true_type{});
        else phase1(std::integral_constant<int, 8>{}, std::false_type{});
      } else if (qm.np == 1) {
        if (full) phase1(std::integral_constant<int, 1>{}, std::true_type{});
        else phase1(std::integral_constant<int, 1>{}, std::false_type{});
      } else {
        if (full) phase1(std::integral_constant<int, 3>{}, std::true_type{});
        else phase1(std::integral_constant<int, 3>{}, std::false_type{});
      }
    } else {
#pragma unroll 4
      for (int i0 = 0; i0 < stage_tok; i0 += kScanNT) {
        if (wn > kCap - kPerBlk) flush();
        const int i = i0 + tid;  // token within the stage
        const bool valid = i < lim;
        float acc[G];
#pragma unroll
        for (int j = 0; j < G; ++j) acc[j] = 0.f;
        if (C8) {
          float x[8];
          Sk::unpack(*reinterpret_cast<const typename Sk::Raw*>(st + (size_t)(i < stage_tok ? i : 0) * rowb), x);
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
          for (int c0 = 0; c0 < C; c0 += 8) sketch_fma8<G, SkBf16>(src[c0 >> 3], qc + c0, C, acc);
        }
        if (edge_stage) {  // NEXT-1: sink / local tokens rank above every score
          const int t = tbase + i;
          if (t < rb.lo || t >= rb.hi) {
#pragma unroll
            for (int j = 0; j < G; ++j) acc[j] = INFINITY;
          }
        }
        bool cand = false;
#pragma unroll
        for (int j = 0; j < G; ++j) cand |= acc[j] >= flo[j];
        cand &= valid;
        const uint32_t cbal = __ballot_sync(0xffffffffu, cand);
        if (cand) {
          const int p = wn + __popc(cbal & lt_mask);
          c_tok[p] = (uint16_t)(cb + i);
          store_scores<G>(c_sc + p * G, acc);
        }
        wn += __popc(cbal);
      }
    }
    // every lane (warp-local staging) / warp is done with the slot before issue() refills it
    if constexpr (kWarpLocal) __syncwarp();
    else __syncthreads();
    slot = slot == kScanStages - 1 ? 0 : slot + 1;
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  flush();
  __syncthreads();
  // ---- the chunk's selection words (sure bits) -> the G rows' bitmaps: every
  // word below N_b is written, so fbm needs no zeroing
  const int nwv = (ntok + 31) >> 5;
  for (int i = tid; i < G * kWords; i += kScanNT) {
    const int j = i / kWords, w = i - j * kWords;
    if (w < nwv) st_keep_u32(fbm + (size_t)(row0 + j) * ldw + (t0 >> 5) + w, s_words[i], pol_keep);
  }
  if (kMma) {
    if (tid < 2) ent_cnt[(creg * 2 + tid) * 2 + sr] = s_bc[tid];  // > kSubCap: overflow (the select's slow path)
    if (half < 0 && tid < 2) ent_cnt[(creg * 2 + tid) * 2 + 1] = 0;  // a whole chunk: empty second sub-region
  } else if (lane == 0) {
    ent_cnt[reg] = wc;
  }
#ifdef SD_SCAN_TRACE
  if (tid == 0) g_scan_trace[blockIdx.y * gridDim.x + blockIdx.x][1] = globaltimer_ns();
#endif
  pdl_launch_dependents();
}

// --------------------------------------------------------------------------- 3. select (per q-head)
// One CTA per row: sure = popcount of the row's fbm words (the scan's sure
// bits), r = k_b - sure; the row's band entries (mask bit j) are gathered into
// shared memory, the exact r-th largest band key tau found by an adaptive radix
// select, exact ties at tau resolved lowest token first, and the band winners
// OR-ed into fbm.  If any check fails (region overflow, band > sel_cap, r < 0
// or r > band, too many ties) the row is recomputed exactly the slow way into
// a zeroed fbm row.
template <int G, class Sk, bool Pair, bool Two>
__global__ void __launch_bounds__(Two ? 2 * kSelNT : kSelNT, Two ? 2 : 4) sbs_select_kernel(const SelArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ SelShared<(Two ? 2 : 1) * kSelNT, Two ? 2 : 1> ush;
  // one CTA per q-row, or per head pair (consecutive heads)
  select_core<G, Sk, Pair, Two>(a, blockIdx.x * (Two ? 2 : 1), smem, ush);
  pdl_launch_dependents();
}

// --------------------------------------------------------------------------- 4. per-head index lists
// Optional (idx_out requested): fbm row -> ascending token list.
constexpr int kIdxNT = 256;
__global__ void __launch_bounds__(kIdxNT) sbs_idx_kernel(const int* __restrict__ seq_lens, int max_len, int Hq,
                                                         const uint32_t* __restrict__ fbm, int ldw,
                                                         int* __restrict__ idx_out, int k_max_out) {
  __shared__ uint32_t warp_tot[33];
  const int row = blockIdx.x, b = row / Hq, tid = threadIdx.x;
  pdl_wait();
  const int N = seq_len_dev(seq_lens, b, max_len);
  const int nw = (max(N, 0) + 31) >> 5;
  const uint32_t* fr = fbm + (size_t)row * ldw;
  int* dst = idx_out + (size_t)row * k_max_out;
  int base = 0;
  for (int w0 = 0; w0 < nw; w0 += kIdxNT) {
    const int w = w0 + tid;
    uint32_t word = w < nw ? fr[w] : 0u;
    uint32_t tot;
    uint32_t p = (uint32_t)base + block_excl_scan<kIdxNT>(__popc(word), warp_tot, &tot);
    while (word) {
      const int bit = __ffs(word) - 1;
      word &= word - 1;
      if (p < (uint32_t)k_max_out) dst[p] = w * 32 + bit;
      ++p;
    }
    base += (int)tot;
  }
}

// --------------------------------------------------------------------------- 5. shard candidates
// Sequence shard: the selection bitmap of every q-row
// of (b, g) -> its candidates in ascending local index order with their fp32
// indexer scores (cand_idx / cand_scores [B*Hq][k_max], -1 / -inf padded).
// G = 4, C = 8, bf16 sketch: a selected token's score is recomputed with the
// scan's MMA on the same 32-token block, so it is the scan's bits.  Grid
// (8192-token tiles, B*Hkv); a tile's output offset per head = the set bits of
// the head's earlier tiles.
constexpr int kEmitNT = 256;
__global__ void __launch_bounds__(kEmitNT) sbs_emit_kernel(
    const void* __restrict__ q, int q_dtype, const uint16_t* __restrict__ sk, const int* __restrict__ channel_ids,
    const int* __restrict__ page_table, const int* __restrict__ seq_lens, int max_len, int max_pages, int Hkv,
    const uint32_t* __restrict__ fbm, int ldw, const int* __restrict__ counts, int* __restrict__ cand_idx,
    float* __restrict__ cand_scores, int k_max) {
  constexpr int G = 4, C = 8, kW = kRangeTok / 32;  // words per tile and head
  static_assert(kW == kEmitNT, "one selection word per thread and head");
  __shared__ uint32_t s_w[G][kW];
  __shared__ int s_pre[G][kW];
  __shared__ int s_wt[G][kEmitNT / 32];
  __shared__ int s_base[G];
  __shared__ float s_qc[G * C];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int bg = blockIdx.y, b = bg / Hkv, g = bg - b * Hkv;
  const int Hq = Hkv * G, row0 = b * Hq + g * G;
  const int tile = blockIdx.x, T0 = tile * kRangeTok;
  pdl_wait();  // the bitmaps and counts come from the select
  const int N = max(0, seq_len_dev(seq_lens, b, max_len));
  if (tile == 0) {  // padding past each row's count
    for (int j = 0; j < G; ++j) {
      const int c = max(0, counts[row0 + j]);
      for (int i = c + tid; i < k_max; i += kEmitNT) {
        cand_idx[(size_t)(row0 + j) * k_max + i] = -1;
        cand_scores[(size_t)(row0 + j) * k_max + i] = -INFINITY;
      }
    }
  }
  if (T0 >= N) return;
  const int nwt = min(kW, (N - T0 + 31) >> 5);
  if (tid < G * C) {
    const int j = tid / C, c = tid - j * C;
    const int ch = __ldg(channel_ids + (size_t)bg * C + c);
    const size_t e = (size_t)(row0 + j) * kD + ch;
    s_qc[tid] = q_dtype == SD_F32 ? reinterpret_cast<const float*>(q)[e] : bf_lo(reinterpret_cast<const uint16_t*>(q)[e]);
  }
  // set bits of the earlier tiles, per head
  int before[G];
#pragma unroll
  for (int j = 0; j < G; ++j) {
    int c = 0;
    const uint32_t* fr = fbm + (size_t)(row0 + j) * ldw;
    for (int w = tid; w < tile * kW; w += kEmitNT) c += __popc(fr[w]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    before[j] = c;
  }
  // this tile's words and their exclusive prefix per head
  int incl[G], cnt[G];
#pragma unroll
  for (int j = 0; j < G; ++j) {
    const uint32_t w = tid < nwt ? fbm[(size_t)(row0 + j) * ldw + (T0 >> 5) + tid] : 0u;
    s_w[j][tid] = w;
    cnt[j] = __popc(w);
    incl[j] = cnt[j];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl[j], o);
      if (lane >= o) incl[j] += y;
    }
    if (lane == 31) s_wt[j][warp] = incl[j];
  }
  __shared__ int s_before[G][kEmitNT / 32];
  if (lane == 0) {
#pragma unroll
    for (int j = 0; j < G; ++j) s_before[j][warp] = before[j];
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < G; ++j) {
    int wb = 0;
    for (int w = 0; w < warp; ++w) wb += s_wt[j][w];
    s_pre[j][tid] = wb + incl[j] - cnt[j];
  }
  if (tid < G) {
    int bb = 0;
    for (int w = 0; w < kEmitNT / 32; ++w) bb += s_before[tid][w];
    s_base[tid] = bb;
  }
  __syncthreads();
  const SkMmaQ qm = sk_mma_q([](int j, int c) { return s_qc[j * C + c]; }, q_dtype == SD_F32 ? 3 : 1);
  const int* pt = page_table + (size_t)b * max_pages;
  const int r = lane >> 2, uu = lane & 3, h0 = 2 * (uu & 1);
  const int tofs = r + ((uu >> 1) << 4);
  // warp per 32-token block (selection word), 4 blocks in flight
  for (int i0 = warp; i0 < nwt; i0 += 4 * (kEmitNT / 32)) {
    uint32_t a[4][4];
    bool any[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int wi = i0 + u * (kEmitNT / 32);
      any[u] = wi < nwt && (s_w[0][wi] | s_w[1][wi] | s_w[2][wi] | s_w[3][wi]) != 0u;
      if (any[u]) {
        const int t0 = T0 + wi * 32;
        sk_mma_a_global(a[u], sk, t0, N,
                        [pt, g, Hkv](int t) { return sketch_row_elem(__ldg(pt + (t >> 4)), t & 15, g, Hkv, C); });
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (!any[u]) continue;
      const int wi = i0 + u * (kEmitNT / 32);
      float d[4];
      sk_mma_score(a[u], qm, d);
#pragma unroll
      for (int x = 0; x < 4; ++x) {
        const int j = h0 + (x & 1), bit = tofs + 8 * (x >> 1);
        const uint32_t w = s_w[j][wi];
        if ((w >> bit) & 1u) {
          const int pos = s_base[j] + s_pre[j][wi] + __popc(w & ((1u << bit) - 1u));
          if (pos < k_max) {
            cand_idx[(size_t)(row0 + j) * k_max + pos] = T0 + wi * 32 + bit;
            cand_scores[(size_t)(row0 + j) * k_max + pos] = d[x];
          }
        }
      }
    }
  }
}

template <class Kern>
cudaError_t set_smem(Kern k, size_t bytes) {
  return ensure_dyn_smem(reinterpret_cast<const void*>(k), bytes);
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

// Shared-memory band capacity of the select kernel.  The band holds the tokens
// between the two sample order statistics: about (2 z sigma + 2) / f tokens
// (sigma = sqrt(k f (1 - f)), f = sample fraction) plus the two edge bins;
// sized at 1.25x that + 1024, within [4096, kSelCap] (4 select CTAs per SM at
// the low end, 1 at the high end).
int band_capacity(int max_seq_len, Budget bud, int sample_nt) {
  const double N = std::max(1, max_seq_len);
  const double NK = bud.kfrom ? std::max(1, bud.max_from) : N;  // sequence shard: k_b from the global length
  const double k = std::min(N, bud.k_fixed > 0 ? std::min<double>(bud.k_fixed, NK)
                               : bud.regions() ? std::max(1.0, bud.heavy_fraction * N + bud.n_sink + bud.n_local)
                                               : std::ceil(NK / bud.S));
  const double f = std::min(1.0, (double)sample_rounds(max_seq_len) * sample_nt * kSampleSlots / N);
  const double sig = std::sqrt(k * f * (1.0 - f));
  // the band spans dr sample ranks; the tokens between two sample order
  // statistics dr ranks apart number dr / f with a relative spread ~ 1 / sqrt(dr)
  const double dr = 2.0 * kBracketZ * sig + 2.0;
  const double band = dr / f;
  const double margin = 1.0 + 4.5 / std::sqrt(std::max(dr, 1.0));
  const int cap = (int)std::min<double>(kSelCap, std::max(4096.0, band * margin + 256.0));
  return (cap + 255) & ~255;
}

template <int G, class Sk>
cudaError_t sbs_launch_t(const Geo& geo, const sd_paged_kv& kv, const sd_sketch& skc, const void* q, Budget bud,
                         const SbsBuffers& w, cudaStream_t st) {
  const void* sk = skc.pages;
  const int C = skc.channels;
  const int BG = geo.B * geo.Hkv;
  cudaError_t e;
  {
    const size_t smem = sizeof(uint32_t) * G * (kHistWords + 512) + sizeof(float) * G * C + (size_t)G * kD * 4 +
                        sizeof(int) * C + sizeof(uint32_t) * G * 32;
    const int snt = sample_threads(BG, geo.max_seq_len, geo.sms);
    // few (b, g) rows: two CTAs per (b, g), half the heads each (fills more SMs)
    constexpr int GH = G >= 2 ? G / 2 : 1;
    const bool split = G >= 2 && snt == kSampleThreads && 2 * BG <= geo.sms;
    const bool multi = sample_rounds(geo.max_seq_len) > 1;
    auto kern = snt == 512 ? sbs_sample_kernel<G, Sk, 512, G, false>
                : split ? (multi ? sbs_sample_kernel<G, Sk, kSampleThreads, GH, true>
                                 : sbs_sample_kernel<G, Sk, kSampleThreads, GH, false>)
                        : (multi ? sbs_sample_kernel<G, Sk, kSampleThreads, G, true>
                                 : sbs_sample_kernel<G, Sk, kSampleThreads, G, false>);
    const size_t smem_used = split ? sizeof(uint32_t) * GH * (kHistWords + 512) + sizeof(float) * GH * C + (size_t)GH * kD * 4 +
                                         sizeof(int) * C + sizeof(uint32_t) * GH * 32
                                   : smem;
    if (SkMma<G, Sk>::value && C == 8) {  // tensor-core sample (the scan's scores)
      const int H = split ? 2 : 4;
      const size_t smem_m = sizeof(uint32_t) * H * (kHistWords + 512) + (size_t)4 * kD * 4 + sizeof(int) * 8 +
                            sizeof(uint32_t) * (H * 32 + 32);  // group sums + 32 dummy words
      auto km = snt == 512 ? sbs_sample_mma_kernel<512, 4, false>
                : split ? (multi ? sbs_sample_mma_kernel<kSampleThreads, 2, true> : sbs_sample_mma_kernel<kSampleThreads, 2, false>)
                        : (multi ? sbs_sample_mma_kernel<kSampleThreads, 4, true> : sbs_sample_mma_kernel<kSampleThreads, 4, false>);
      e = set_smem(km, smem_m);
      if (e != cudaSuccess) return e;
      e = launch_pdl(km, dim3(split ? 2 * BG : BG), dim3(snt), smem_m, st, true, q, geo.kv_dtype,
                     reinterpret_cast<const uint16_t*>(sk), skc.channel_ids, kv.page_table, kv.seq_lens, geo.max_seq_len,
                     geo.max_pages, geo.Hkv, bud.dev(), w.thr, w.counters);
    } else {
      e = set_smem(kern, smem_used);
      if (e != cudaSuccess) return e;
      e = launch_pdl(kern, dim3(split ? 2 * BG : BG), dim3(snt), smem_used, st, true, q, geo.kv_dtype, sk, skc.channel_ids, C,
                     kv.page_table, kv.seq_lens, geo.max_seq_len, geo.max_pages, geo.Hkv, bud.dev(), w.thr, w.counters);
    }
    if (e != cudaSuccess) return e;
    if (w.ev) cudaEventRecord(w.ev[0], st);
  }
  const int nch = (geo.max_seq_len + kRangeTok - 1) / kRangeTok;
  const int sel_cap = band_capacity(geo.max_seq_len, bud, sample_threads(BG, geo.max_seq_len, geo.sms));
  const bool pair = (SkMma<G, Sk>::value || SkMmaF8<G, Sk>::value) && C == 8;  // the tensor-core scan's pair regions
  // the region count table: every band region of the longest row, unless the
  // select's shared memory cannot hold it (those rows take the exact slow path)
  // (the pair regions' counts are read straight from global memory: no table)
  int nreg_cap = pair ? 0 : nch * kScanWarps;
  if (sel_core_smem(1, sel_cap, C, nreg_cap) + sizeof(SelShared<kSelNT, 1>) + 1024 > 227 * 1024) nreg_cap = 0;
  SelArgs sa{q, geo.kv_dtype, sk, skc.channel_ids, C, kv.page_table, kv.seq_lens, geo.max_seq_len, geo.max_pages,
             geo.Hkv, bud.dev(), w.thr, w.ent_tok, w.ent_sc, w.ent_cnt, nch, w.fbm, w.ldw, w.scratch, w.ld,
             w.counts_out, w.force_fallback, w.err, sel_cap, nreg_cap};
  {
    // 4 CTAs/SM (NS = 2) when the grid exceeds one 3-CTA/SM wave
    const int ns = (size_t)nch * BG > (size_t)3 * geo.sms ? 2 : 3;
    const size_t smem = (size_t)ns * kScanStageTok8 * 16 +
                        sizeof(float) * G * C + sizeof(int) * (kRangeTok / 16) + sizeof(uint32_t) * G * (kRangeTok / 32) +
                        (sizeof(float) * G + 2 * sizeof(uint16_t)) * kScanWarps * scan_cand_cap(ns);
    // the final 4-CTA/SM wave's worth of items as half-chunk CTAs (tensor-core
    // pair-region path only): the scan's tail is half as long
    const int n_items = nch * BG;
    const int n_half = (pair && ns == 2) ? std::min(n_items / 4, (SD_SCAN_HALF * geo.sms) / 2) : 0;
    dim3 grid(n_items + n_half);
    // the fp8 sketch is C = 8 only (host-checked): no generic-C fp8 variant
    auto kern = C == 8 ? (ns == 2 ? sbs_scan_kernel<G, true, Sk, 2> : sbs_scan_kernel<G, true, Sk, 3>)
                       : (ns == 2 ? sbs_scan_kernel<G, false, SkBf16, 2> : sbs_scan_kernel<G, false, SkBf16, 3>);
    e = set_smem(kern, smem);
    if (e != cudaSuccess) return e;
    e = launch_pdl(kern, grid, dim3(kScanNT), smem, st, true, q, geo.kv_dtype,
                   reinterpret_cast<const char*>(skc.pages), skc.channel_ids, C, kv.page_table, kv.seq_lens,
                   geo.max_seq_len, geo.max_pages, geo.Hkv, (const uint32_t*)w.thr, w.ent_tok, w.ent_sc, w.ent_cnt, w.fbm, w.ldw, nch,
                   bud.dev(), n_half);
    if (e != cudaSuccess) return e;
    if (w.ev) cudaEventRecord(w.ev[1], st);
  }
  {
    // two heads per CTA when that still fits 2 CTAs per SM (B*Hq/2 pairs in one wave)
    const bool two = pair && sel_core_smem(2, sel_cap, C, nreg_cap) + sizeof(uint32_t) * 2 * kHistWords + 4096 <= 113 * 1024;
    const size_t smem = sel_core_smem(two ? 2 : 1, sel_cap, C, nreg_cap);
    auto kern = two ? sbs_select_kernel<G, Sk, true, true>
                    : pair ? sbs_select_kernel<G, Sk, true, false> : sbs_select_kernel<G, Sk, false, false>;
    e = set_smem(kern, smem);
    if (e != cudaSuccess) return e;
    e = launch_pdl(kern, dim3(geo.B * geo.Hq / (two ? 2 : 1)), dim3(two ? 2 * kSelNT : kSelNT), smem, st, true, sa);
    if (e != cudaSuccess) return e;
  }
  if (w.ev) cudaEventRecord(w.ev[2], st);
  return cudaSuccess;
}

}  // namespace

cudaError_t launch_sbs_emit(const Geo& g, const sd_paged_kv& kv, const sd_sketch& sk, const void* q,
                            const SbsBuffers& w, int* cand_idx, float* cand_scores, int k_max, cudaStream_t st) {
  if (g.G != 4 || sk.channels != 8 || sk.dtype != SD_BF16) return cudaErrorInvalidValue;
  const int nch = (g.max_seq_len + kRangeTok - 1) / kRangeTok;
  return launch_pdl(sbs_emit_kernel, dim3(nch, g.B * g.Hkv), dim3(kEmitNT), 0, st, true, q, g.kv_dtype,
                    reinterpret_cast<const uint16_t*>(sk.pages), sk.channel_ids, kv.page_table, kv.seq_lens,
                    g.max_seq_len, g.max_pages, g.Hkv, (const uint32_t*)w.fbm, w.ldw, (const int*)w.counts_out,
                    cand_idx, cand_scores, k_max);
}

cudaError_t launch_sbs_select(const Geo& g, const sd_paged_kv& kv, const sd_sketch& sk, const void* q, Budget bud,
                              const SbsBuffers& w, cudaStream_t st) {
  cudaError_t e;
  switch (g.G) {
    case 1: e = sk.dtype == SD_E4M3 ? sbs_launch_t<1, SkE4m3>(g, kv, sk, q, bud, w, st)
                                      : sbs_launch_t<1, SkBf16>(g, kv, sk, q, bud, w, st); break;
    case 2: e = sk.dtype == SD_E4M3 ? sbs_launch_t<2, SkE4m3>(g, kv, sk, q, bud, w, st)
                                      : sbs_launch_t<2, SkBf16>(g, kv, sk, q, bud, w, st); break;
    case 4: e = sk.dtype == SD_E4M3 ? sbs_launch_t<4, SkE4m3>(g, kv, sk, q, bud, w, st)
                                      : sbs_launch_t<4, SkBf16>(g, kv, sk, q, bud, w, st); break;
    case 8: e = sk.dtype == SD_E4M3 ? sbs_launch_t<8, SkE4m3>(g, kv, sk, q, bud, w, st)
                                      : sbs_launch_t<8, SkBf16>(g, kv, sk, q, bud, w, st); break;
    default: return cudaErrorInvalidValue;
  }
  if (e != cudaSuccess || !w.idx_out) return e;
  return launch_pdl(sbs_idx_kernel, dim3(g.B * g.Hq), dim3(kIdxNT), 0, st, true, kv.seq_lens, g.max_seq_len, g.Hq,
                    (const uint32_t*)w.fbm, w.ldw, w.idx_out, w.k_max_out);
}

}  // namespace sd

#ifdef SD_SCAN_TRACE
extern "C" int sd_debug_scan_trace(unsigned long long* host, int n_ctas) {
  return (int)cudaMemcpyFromSymbol(host, sd::g_scan_trace, sizeof(unsigned long long) * 2 * n_ctas);
}
#endif
