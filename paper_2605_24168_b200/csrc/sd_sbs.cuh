// sd_sbs.cuh - data contract of the fused "sample-bracket select" (SBS) path
// between the selection kernels (k_fused.cu) and the gather-attend kernels
// (k_rows_mma.cu, k_rows.cu).
//
// Per q-row (b, h) with N_b tokens:
//   thr[row] = {lo, hi, flo, fsure}  sample bracket keys + the equivalent fp32
//                                    thresholds for the scan        (sbs_sample_kernel)
//   fbm[row][t / 32] bit t = key(s_t) > hi after sbs_scan_kernel (sure tokens),
//                          = t is in the exact top-k_b after sbs_select_kernel
//   band entries (lo <= key <= hi for some head of the group): token | head
//   mask << 24 and the scores.  Tensor-core scan (G = 4, C = 8): one region per
//   (b, g, 8192-token chunk, head pair p) of capacity 8 * band_region_cap(4),
//   filled by the scan CTA's 8 warps through a shared-memory position counter,
//   the pair's 2 scores per entry (mask bits 2p, 2p + 1); its two halves are
//   sub-regions with a count each (the scan's last items run as two half-chunk
//   CTAs, one per sub-region; a whole-chunk CTA fills sub-region 0).  Otherwise: one region
//   per (b, g, chunk, scan warp) of capacity band_region_cap(G), G scores per entry.
// where key() is the order-preserving uint32 map of the fp32 indexer score
// (sd_common.cuh score_key).  A gather-attend CTA owning tokens [T0, T1) of
// (b, g) ORs the G heads' fbm words of its range into the ascending GQA union
// rows; the per-head bits give each row's head mask.
#pragma once
#include "sd_common.cuh"

namespace sd {

constexpr int kRangeTok = 8192;  // tokens per scan CTA and per gather-attend CTA

}  // namespace sd

namespace sd {

// Union-row helpers for a gather-attend CTA owning tokens [T0, T1) of (b, g):
// bm[G][nw] holds the G heads' selection words of the range, upre[w] =
// exclusive prefix of popc(OR of the G words) (upre[nw] = row count).

// Load the range's words and build upre; returns the union row count.
// All threads must call it.
template <int G, int NT>
__device__ __forceinline__ int union_prologue(const uint32_t* __restrict__ fbm, int ldw, int row0, int T0, int T1,
                                              uint32_t* bm, int* upre, int* warp_tot) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nw = (T1 - T0 + 31) >> 5;
  for (int i = tid; i < G * nw; i += NT) {
    const int j = i / nw, w = i - j * nw;
    bm[i] = fbm[(size_t)(row0 + j) * ldw + (T0 >> 5) + w];
  }
  __syncthreads();
  int base = 0;
  for (int w0 = 0; w0 < nw; w0 += NT) {
    const int w = w0 + tid;
    uint32_t u = 0;
    if (w < nw) {
#pragma unroll
      for (int j = 0; j < G; ++j) u |= bm[j * nw + w];
    }
    const int c = __popc(u);
    int x = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[warp] = x;
    __syncthreads();
    int wb = 0, all = 0;
#pragma unroll
    for (int i = 0; i < NT / 32; ++i) {
      const int t = warp_tot[i];
      if (i < warp) wb += t;
      all += t;
    }
    if (w < nw) upre[w] = base + wb + x - c;
    base += all;
    __syncthreads();
  }
  if (tid == 0) upre[nw] = base;
  __syncthreads();
  return base;
}

// Token offset (t - T0) of union row i (0 <= i < upre[nw]).
template <int G>
__device__ __forceinline__ int union_row_token(const uint32_t* bm, const int* upre, int nw, int i) {
  int lo = 0, hi = nw - 1;  // largest w with upre[w] <= i and a set bit
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (upre[mid] <= i) lo = mid;
    else hi = mid - 1;
  }
  // words with no set bits share upre with the next word; the largest such w
  // with upre[w] <= i is the one holding row i
  uint32_t word = 0;
#pragma unroll
  for (int j = 0; j < G; ++j) word |= bm[j * nw + lo];
  int n = i - upre[lo], pos = 0;  // n-th (0-based) set bit of word
#pragma unroll
  for (int w = 16; w >= 1; w >>= 1) {
    const int c = __popc(word & ((1u << w) - 1u));
    if (n >= c) {
      n -= c;
      pos += w;
      word >>= w;
    }
  }
  return lo * 32 + pos;
}

}  // namespace sd
