// sd_select.cuh - block-wide exact selection primitives (A3).
//
// radix_select_block: over n order-preserving uint32 keys produced by a
// functor, find the k-th largest key tau and need_eq = how many keys equal to
// tau belong to the top k (the remaining top-k keys are exactly those > tau).
// Three histogram passes of 11/11/10 bits in shared memory.
//
// emit_block: walk the keys in index order and compact the selected ones
// (key > tau, or key == tau and among the first need_eq such keys in index
// order, S:200 tie rule) with block-wide prefix scans -> ascending output.
#pragma once
#include "sd_common.cuh"

namespace sd {

template <int NT>
struct SelectSmem {
  uint32_t hist[2048];
  uint32_t warp_tot[33];
  uint32_t digit, kr;
};

// Exclusive block scan of one value per thread (NT threads, NT % 32 == 0).
template <int NT>
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* warp_tot, uint32_t* total) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[w] = x;
  __syncthreads();
  if (w == 0) {
    uint32_t t = lane < NW ? warp_tot[lane] : 0u;
    uint32_t z = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, z, o);
      if (lane >= o) z += y;
    }
    if (lane < NW) warp_tot[lane] = z - t;
    if (lane == 31) warp_tot[32] = z;
  }
  __syncthreads();
  const uint32_t r = warp_tot[w] + x - v;
  *total = warp_tot[32];
  __syncthreads();
  return r;
}

// KeyAt(i) -> uint32 key for i in [0, n).  Requires 1 <= k <= n.
template <int NT, class KeyAt>
__device__ __forceinline__ void radix_select_block(KeyAt key_at, int n, uint32_t k, SelectSmem<NT>& sm,
                                                   uint32_t* tau_out, uint32_t* need_eq_out) {
  const int tid = threadIdx.x;
  uint32_t prefix = 0, pmask = 0, kr = k;
#pragma unroll 1
  for (int pass = 0; pass < 3; ++pass) {
    const int shift = pass == 0 ? 21 : (pass == 1 ? 10 : 0);
    const int nb = pass == 2 ? 1024 : 2048;
    for (int i = tid; i < 2048; i += NT) sm.hist[i] = 0;
    __syncthreads();
    for (int i = tid; i < n; i += NT) {
      const uint32_t key = key_at(i);
      if ((key & pmask) == prefix) atomicAdd(&sm.hist[(key >> shift) & (nb - 1)], 1u);
    }
    __syncthreads();
    // thread tid owns `per` consecutive bins, highest bins first
    const int per = (nb + NT - 1) / NT;
    uint32_t local = 0;
    for (int j = 0; j < per; ++j) {
      const int bin = nb - 1 - (tid * per + j);
      if (bin >= 0) local += sm.hist[bin];
    }
    uint32_t tot;
    uint32_t above = block_excl_scan<NT>(local, sm.warp_tot, &tot);
    for (int j = 0; j < per; ++j) {
      const int bin = nb - 1 - (tid * per + j);
      if (bin < 0) break;
      const uint32_t c = sm.hist[bin];
      if (above < kr && above + c >= kr) { sm.digit = (uint32_t)bin; sm.kr = kr - above; }
      above += c;
    }
    __syncthreads();
    prefix |= sm.digit << shift;
    pmask |= (uint32_t)(nb - 1) << shift;
    kr = sm.kr;
    __syncthreads();
  }
  *tau_out = prefix;
  *need_eq_out = kr;
}

// Emit, in increasing i, every selected i: key > tau, or key == tau and among
// the first need_eq (counting eq_offset ties that precede this range).
// Emit(pos, i, key) is called once per selected element with its output slot.
// Returns the number emitted (block-uniform).
template <int NT, int ITEMS, class KeyAt, class Emit>
__device__ __forceinline__ uint32_t emit_block(KeyAt key_at, int n, uint32_t tau, uint32_t need_eq,
                                               uint32_t eq_offset, SelectSmem<NT>& sm, Emit emit,
                                               uint32_t* eq_seen = nullptr) {
  const int tid = threadIdx.x;
  uint32_t run_sel = 0, run_eq = eq_offset;
  for (int tile = 0; tile < n; tile += NT * ITEMS) {
    const int base = tile + tid * ITEMS;
    uint32_t gt = 0, eq = 0;
    uint32_t keys[ITEMS];
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) {
      const int i = base + j;
      keys[j] = 0;
      if (i < n) {
        keys[j] = key_at(i);
        gt |= (uint32_t)(keys[j] > tau) << j;
        eq |= (uint32_t)(keys[j] == tau) << j;
      }
    }
    uint32_t eq_tot;
    const uint32_t eq_before = run_eq + block_excl_scan<NT>(__popc(eq), sm.warp_tot, &eq_tot);
    uint32_t sel = gt, e_seen = 0;
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) {
      if ((eq >> j) & 1u) {
        if (eq_before + e_seen < need_eq) sel |= 1u << j;
        ++e_seen;
      }
    }
    uint32_t sel_tot;
    uint32_t pos = run_sel + block_excl_scan<NT>(__popc(sel), sm.warp_tot, &sel_tot);
#pragma unroll
    for (int j = 0; j < ITEMS; ++j)
      if ((sel >> j) & 1u) emit(pos++, base + j, keys[j]);
    run_eq += eq_tot;
    run_sel += sel_tot;
  }
  if (eq_seen) *eq_seen = run_eq - eq_offset;
  return run_sel;
}

}  // namespace sd
