// k_attend_pk.cu - persistent gather-attend over the GQA union rows of the
// fused path (A4/A5 of SURVEY.md 8(a); P:255 per-head index sets; "the KV
// cache's vector dimension provides sufficient contiguous memory").
//
// Memory-latency view.  The rows are gathered with 16-B cp.async into a
// shared-memory ring; at ~6.5 TB/s and a few microseconds of loaded DRAM
// latency an SM needs >100 KB of copies in flight.  A CTA per 8192-token range
// (k_rows_mma.cu) holds only ~600 rows at N = 128K, S = 50: its ring drains at
// the end of every range and refills only after the next CTA's prologue.
// Here two CTAs per SM, warp-specialised (attend_union_ws_kernel below), loop
// over work units; the producers' issue cursor runs ahead across unit and item
// boundaries, so copies stay in flight while a unit ends and the next starts.
//
// Work unit = up to kPkBatch consecutive union rows of one item, item = one
// 8192-token range of one (b, g); a CTA's first item is blockIdx.x, the rest
// are claimed one item ahead from an atomic counter (zeroed by
// sbs_sample_kernel).  The producers resolve the NEXT unit (selection words ->
// ascending union rows -> K/V row index + head mask, page ids in registers)
// into the other half of a double buffer while the consumers work on the
// current one.
//
// Per 64-row stage each consumer warp runs its 16-row tile on the tensor cores
// (mma.sync m16n8k16 bf16 -> fp32): S = Q K^T, masked online softmax,
// O += (P_hi + P_lo) V; the arithmetic is that of attend_rows_mma_kernel.
// At an item's last unit the 4 consumer warps' states are merged (scratch: the
// ring slot just consumed, released to the producers only after the merge)
// into the item's split partial; merge_parts_kernel (PDL) merges the splits in
// split order (deterministic) into out / lse.  Folding that merge into the
// last CTA of each (b, g) needs a gpu-scope fence per item (MEMBAR.ALL.GPU +
// CCTL.IVALL), which drains the in-flight copies: measured 122 -> 240 us at
// cfg3 (barrier-synchronised version).
#include "sd_common.cuh"
#include "sd_internal.h"
#include "sd_sbs.cuh"

namespace sd {
namespace {

constexpr int kPkWarps = 4;
constexpr int kPkThreads = kPkWarps * 32;
constexpr int kPkTile = 16;
constexpr int kPkStageRows = kPkWarps * kPkTile;          // 64
constexpr int kPkRowB = 256;
constexpr int kPkStageBytes = kPkStageRows * 2 * kPkRowB;  // 32 KB: K block then V block
constexpr int kPkStages = 3;
constexpr int kPkBatch = 1024;                            // union rows per work unit
constexpr int kPkItemTok = kRangeTok;                     // 8192 tokens per item
static_assert(kPkItemTok / 32 == 2 * kPkThreads, "two selection words per thread");


__device__ __forceinline__ void cp_async16_pk(uint32_t dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(valid ? 16 : 0) : "memory");
}
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
// D = A(16x16, row; rows 8..15 zero) * B(16x8, col) + D
__device__ __forceinline__ void mma_bf16(float* d, uint32_t a0, uint32_t a2, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(0u), "r"(a2), "r"(0u), "r"(b0), "r"(b1));
}
// D = A(16x16, row) * B(16x8, col) + D with all four A registers
__device__ __forceinline__ void mma_bf16_full(float* d, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                              uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
__device__ __forceinline__ float bf16_round(float x) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r << 16);
}
__device__ __forceinline__ uint32_t swz(int r, int c) { return (uint32_t)(r * kPkRowB + ((c ^ (r & 7)) << 4)); }

// ---------------------------------------------------------------------------
// Warp-specialised variant (default): 8 warps per CTA, 2 CTAs per SM.
// Warps 4-7 (producers, 56 registers after setmaxnreg.dec) resolve work units
// and stream their K/V rows into the ring with cp.async, signalling each stage
// on full[slot] with cp.async.mbarrier.arrive.noinc (the arrive fires when the
// thread's copies have landed); warps 0-3 (consumers, 200 registers) wait on
// full[slot], compute, and release the slot on empty[slot].  Units are handed
// over through double-buffered row lists with ready[buf] / freed[buf]
// mbarriers.  No CTA-wide barrier in the steady state: the copy issue never
// waits for the compute (tools/gather_ws.cu: 6.0 TB/s vs 5.5 TB/s for the
// barrier-synchronised ring at this shape).
constexpr int kWsThreads = 256;
constexpr int kWsConsRegs = 200, kWsProdRegs = 56;

template <int G>
struct WsSmem {
  unsigned char ring[kPkStages][kPkStageBytes];
  uint32_t rowi[2][kPkBatch];
  uint8_t rmask[2][kPkBatch];
  uint16_t qs[2][G * kD];
  int u_it[2], u_nrows[2], u_last[2], u_r0[2];
  int wtot[kPkWarps];
  int next_it;  // dynamically claimed next item (producers)
  uint64_t full[kPkStages], empty[kPkStages], ready[2], freed[2];
};

__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void cp_async_arrive_noinc(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

#ifdef SD_ATTEND_TRACE
// debug builds only (-DSD_ATTEND_TRACE, scripts/attend_trace.py): per CTA
// {start, first unit ready, end, units} in %globaltimer ns
__device__ unsigned long long g_attend_trace[1024][4];
#endif

template <int G>
__global__ void __launch_bounds__(kWsThreads, 2) attend_union_ws_kernel(
    const uint16_t* __restrict__ q, const char* __restrict__ kp, const char* __restrict__ vp,
    const int* __restrict__ page_table, const int* __restrict__ seq_lens, int max_len, int max_pages, int Hkv,
    const uint32_t* __restrict__ fbm, int ldw, float scale_log2, float* __restrict__ part, int splits, int n_items,
    int* __restrict__ work) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  WsSmem<G>& sm = *reinterpret_cast<WsSmem<G>*>(smem_raw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int Hq = Hkv * G;
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < kPkStages; ++s) {
      mbar_init(&sm.full[s], kPkThreads);  // one noinc arrive per producer thread
      mbar_init(&sm.empty[s], kPkWarps);   // one arrive per consumer warp
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&sm.ready[b], 1);
      mbar_init(&sm.freed[b], kPkWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if ((int)blockIdx.x >= n_items) {
    pdl_launch_dependents();
    return;
  }
  pdl_wait();  // selection bitmaps come from sbs_select_kernel
#ifdef SD_ATTEND_TRACE
  if (tid == 0) g_attend_trace[blockIdx.x][0] = globaltimer_ns();
#endif

  if (warp >= kPkWarps) {
    // =================================================================== producers
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kWsProdRegs));
    const int pt_ = tid - kPkThreads, pw = pt_ >> 5;  // producer thread / warp index
    struct ItemRegs {
      int it, N;
      uint2 wv[G];
      int pv[4];
      uint4 qv;
    };
    auto load_item = [&](ItemRegs& r, int it) {
      r.it = it;
      if (it >= n_items) return;
      const int bg = it / splits, split = it - bg * splits;
      const int b = bg / Hkv, g = bg - b * Hkv;
      r.N = max(0, seq_len_dev(seq_lens, b, max_len));  // out of range: an empty row (the select reports)
      const int t0 = split * kPkItemTok;
      const int w0 = (t0 >> 5) + 2 * pt_;
#pragma unroll
      for (int j = 0; j < G; ++j)
        r.wv[j] = w0 < ldw ? *reinterpret_cast<const uint2*>(fbm + (size_t)(b * Hq + g * G + j) * ldw + w0)
                           : make_uint2(0u, 0u);
      const int p0 = (t0 >> 4) + 4 * pt_;
      const int* pt = page_table + (size_t)b * max_pages;
#pragma unroll
      for (int k = 0; k < 4; ++k) r.pv[k] = p0 + k < max_pages ? __ldg(pt + p0 + k) : 0;
      if (pt_ < G * 16)
        r.qv = *reinterpret_cast<const uint4*>(q + (size_t)(b * Hq + g * G + (pt_ >> 4)) * kD + (pt_ & 15) * 8);
    };
    // rows [r0, r0 + kPkBatch) of the item in r -> buffer buf; returns the
    // item's union row count (producer threads only, 2 named barriers)
    auto resolve = [&](const ItemRegs& r, int r0, int buf) -> int {
      const int it = r.it;
      const int bg = it / splits, split = it - bg * splits;
      const int g = bg - (bg / Hkv) * Hkv;
      const int T0 = min(r.N, split * kPkItemTok), ntok = min(r.N, T0 + kPkItemTok) - T0;
      const int nw = (ntok + 31) >> 5;
      const int w0 = 2 * pt_;
      if (r0 == 0 && pt_ < G * 16) *reinterpret_cast<uint4*>(&sm.qs[buf][(pt_ >> 4) * kD + (pt_ & 15) * 8]) = r.qv;
      uint32_t u0 = 0, u1 = 0;
#pragma unroll
      for (int j = 0; j < G; ++j) {
        u0 |= w0 < nw ? r.wv[j].x : 0u;
        u1 |= w0 + 1 < nw ? r.wv[j].y : 0u;
      }
      const int cnt = __popc(u0) + __popc(u1);
      int incl = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      if (lane == 31) sm.wtot[pw] = incl;
      named_sync(1, kPkThreads);
      int pos = incl - cnt, total = 0;
#pragma unroll
      for (int w = 0; w < kPkWarps; ++w) {
        const int t = sm.wtot[w];
        pos += w < pw ? t : 0;
        total += t;
      }
      if (pos < r0 + kPkBatch && pos + cnt > r0) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          uint32_t x = e ? u1 : u0;
          while (x) {
            const int bit = __ffs(x) - 1;
            x &= x - 1;
            if (pos >= r0 && pos < r0 + kPkBatch) {
              uint32_t mk = 0;
#pragma unroll
              for (int j = 0; j < G; ++j) {
                const uint32_t wj = e ? (w0 + 1 < nw ? r.wv[j].y : 0u) : (w0 < nw ? r.wv[j].x : 0u);
                mk |= ((wj >> bit) & 1u) << j;
              }
              const int pg = bit < 16 ? r.pv[2 * e] : r.pv[2 * e + 1];
              sm.rowi[buf][pos - r0] = (uint32_t)(pg * kPS + (bit & 15)) * (uint32_t)Hkv + g;
              sm.rmask[buf][pos - r0] = (uint8_t)mk;
            }
            ++pos;
          }
        }
      }
      named_sync(1, kPkThreads);  // wtot reusable; the buffer is complete
      return total;
    };
    // hand unit u (item it, rows [r0, r0 + nrows), last-of-item flag) to the consumers
    auto publish = [&](int u, int it, int r0, int nrows, int last) {
      const int buf = u & 1;
      if (pt_ == 0) {
        sm.u_it[buf] = it;
        sm.u_r0[buf] = r0;
        sm.u_nrows[buf] = nrows;
        sm.u_last[buf] = last;
        mbar_arrive(&sm.ready[buf]);  // release: the row lists and queries above are visible
      }
    };
    const int ic16 = pt_ & 15, ir0 = pt_ >> 4;
    const char* kpc = kp + ic16 * 16;
    const char* vpc = vp + ic16 * 16;
    int issued = 0;
    auto issue = [&](int buf, int stage, int nrows) {
      const int slot = issued % kPkStages;
      if (issued >= kPkStages) mbar_wait(&sm.empty[slot], (uint32_t)((issued / kPkStages) - 1) & 1u);
      const uint32_t kd = smem_u32(&sm.ring[slot][0]);
      const uint32_t vd = kd + kPkStageRows * kPkRowB;
      const int R0 = stage * kPkStageRows;
      const int nr = min(kPkStageRows, nrows - R0);
      const int nr16 = (nr + 15) & ~15;  // rows of partial tiles are zero-filled
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int rr = ir0 + 8 * i;
        if (rr < nr16) {
          const bool valid = rr < nr;
          const size_t off = valid ? (size_t)sm.rowi[buf][R0 + rr] * kPkRowB : 0;
          const uint32_t d = (uint32_t)(rr * kPkRowB + ((ic16 ^ (rr & 7)) << 4));
          cp_async16_pk(kd + d, kpc + off, valid);
          cp_async16_pk(vd + d, vpc + off, valid);
        }
      }
      cp_async_arrive_noinc(&sm.full[slot]);
      ++issued;
    };

    // items: blockIdx.x first, then claimed from the work counter (zeroed by
    // sbs_sample_kernel) one item ahead, so faster CTAs take more items
    auto claim = [&]() {
      if (pt_ == 0) sm.next_it = gridDim.x + atomicAdd(work, 1);
      named_sync(1, kPkThreads);
      return sm.next_it;
    };
    ItemRegs cur_r, nxt_r;
    int it_c = blockIdx.x, r0_c = 0;
    load_item(cur_r, it_c);
    int total_c = resolve(cur_r, 0, 0);
    load_item(nxt_r, claim());
    int u = 0;
    int nrows_c = min(kPkBatch, total_c);
    publish(0, it_c, 0, nrows_c, r0_c + kPkBatch >= total_c);
    for (;;) {
      const int buf = u & 1;
      const int nst = max(1, (nrows_c + kPkStageRows - 1) / kPkStageRows);
      for (int s = 0; s < nst; ++s) issue(buf, s, nrows_c);
      // next unit: the rest of this item, or the next item
      int it_n, r0_n;
      if (r0_c + kPkBatch < total_c) {
        it_n = it_c;
        r0_n = r0_c + kPkBatch;
      } else {
        it_n = nxt_r.it;
        r0_n = 0;
      }
      const int nb = buf ^ 1;
      if (u >= 1) mbar_wait(&sm.freed[nb], (uint32_t)(((u + 1) >> 1) - 1) & 1u);  // consumers done with unit u - 1
      if (it_n >= n_items) {
        publish(u + 1, n_items, 0, 0, 0);  // end marker
        break;
      }
      int total_n;
      if (r0_n) {
        total_n = resolve(cur_r, r0_n, nb);
      } else {
        total_n = resolve(nxt_r, 0, nb);
        cur_r = nxt_r;
        load_item(nxt_r, claim());
      }
      const int nrows_n = min(kPkBatch, total_n - r0_n);
      publish(u + 1, it_n, r0_n, nrows_n, r0_n + kPkBatch >= total_n);
      it_c = it_n;
      r0_c = r0_n;
      total_c = total_n;
      nrows_c = nrows_n;
      ++u;
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
  } else {
    // =================================================================== consumers
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kWsConsRegs));
    const int qr = lane >> 2, qc2 = (lane & 3) * 2;
    const int lr = lane & 7, lm = lane >> 3;
    uint32_t qa0[8], qa2[8];
    float oT[8][4];
    float m = -INFINITY, lsum = 0.f;
    int consumed = 0;
    for (int u = 0;; ++u) {
      const int buf = u & 1;
      mbar_wait(&sm.ready[buf], (uint32_t)(u >> 1) & 1u);
      const int it_c = sm.u_it[buf];
#ifdef SD_ATTEND_TRACE
      if (tid == 0 && u == 0) g_attend_trace[blockIdx.x][1] = globaltimer_ns();
      if (tid == 0 && it_c >= n_items) {
        g_attend_trace[blockIdx.x][2] = globaltimer_ns();
        g_attend_trace[blockIdx.x][3] = (unsigned long long)u;
      }
#endif
      if (it_c >= n_items) break;
      const int r0_c = sm.u_r0[buf], nrows_c = sm.u_nrows[buf], last_c = sm.u_last[buf];
      if (r0_c == 0) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          qa0[kk] = qa2[kk] = 0u;
          if (qr < G) {
            const uint16_t* qrow = &sm.qs[buf][qr * kD + kk * 16 + qc2];
            qa0[kk] = *reinterpret_cast<const uint32_t*>(qrow);
            qa2[kk] = *reinterpret_cast<const uint32_t*>(qrow + 8);
          }
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) oT[i][0] = oT[i][1] = oT[i][2] = oT[i][3] = 0.f;
        m = -INFINITY;
        lsum = 0.f;
      }
      const int nst = max(1, (nrows_c + kPkStageRows - 1) / kPkStageRows);
      int slot = 0;
      for (int cc = 0; cc < nst; ++cc) {
        slot = consumed % kPkStages;
        mbar_wait(&sm.full[slot], (uint32_t)(consumed / kPkStages) & 1u);
        const unsigned char* st = sm.ring[slot];
        const uint8_t* msk = sm.rmask[buf] + cc * kPkStageRows;
        const int nr = min(kPkStageRows, nrows_c - cc * kPkStageRows);
        const int trow = warp * kPkTile;
        if (trow < nr) {
          const uint32_t kb = smem_u32(st) + trow * kPkRowB;
          const uint32_t vb = smem_u32(st + kPkStageRows * kPkRowB) + trow * kPkRowB;
          float sc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const int r = (lm >> 1) * 8 + lr, c = 2 * kk + (lm & 1);
            uint32_t b0, b1, b2, b3;
            ldsm_x4(kb + swz(r, c), b0, b1, b2, b3);
            mma_bf16(sc[0], qa0[kk], qa2[kk], b0, b1);
            mma_bf16(sc[1], qa0[kk], qa2[kk], b2, b3);
          }
          float x[4];
#pragma unroll
          for (int nt = 0; nt < 2; ++nt) {
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int rr = trow + nt * 8 + qc2 + e;
              const bool ok = qr < G && rr < nr && ((msk[rr] >> qr) & 1u);
              x[nt * 2 + e] = ok ? sc[nt][e] * scale_log2 : -INFINITY;
            }
          }
          float tmax = fmaxf(fmaxf(x[0], x[1]), fmaxf(x[2], x[3]));
          tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 1));
          tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 2));
          const bool grow = tmax > m;
          if (__any_sync(0xffffffffu, grow)) {
            const float mn = grow ? tmax : m;
            const float corr = (m == -INFINITY) ? 0.f : exp2f(m - mn);
            lsum *= corr;
            const float ca = __shfl_sync(0xffffffffu, corr, (lane & 3) * 8);
            const float cb = __shfl_sync(0xffffffffu, corr, (lane & 3) * 8 + 4);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              oT[i][0] *= ca;
              oT[i][1] *= cb;
              oT[i][2] *= ca;
              oT[i][3] *= cb;
            }
            m = mn;
          }
          float p[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) p[i] = (x[i] == -INFINITY) ? 0.f : exp2f(x[i] - m);
          lsum += (p[0] + p[1]) + (p[2] + p[3]);
          const uint32_t ph0 = pack_bf16(p[0], p[1]), ph2 = pack_bf16(p[2], p[3]);
          const uint32_t pl0 = pack_bf16(p[0] - bf16_round(p[0]), p[1] - bf16_round(p[1]));
          const uint32_t pl2 = pack_bf16(p[2] - bf16_round(p[2]), p[3] - bf16_round(p[3]));
#pragma unroll
          for (int mt = 0; mt < 8; ++mt) {
            const int r = (lm >> 1) * 8 + lr, c = 2 * mt + (lm & 1);
            uint32_t a0, a1, a2, a3;
            ldsm_x4_t(vb + swz(r, c), a0, a1, a2, a3);
            mma_bf16_full(oT[mt], a0, a1, a2, a3, ph0, ph2);
            mma_bf16_full(oT[mt], a0, a1, a2, a3, pl0, pl2);
          }
        }
        ++consumed;
        __syncwarp();
        // the item's last slot is kept as merge scratch until the merge is done
        if (!(last_c && cc == nst - 1) && lane == 0) mbar_arrive(&sm.empty[slot]);
      }
      // this unit's row masks and queries are read: the buffer may be refilled
      if (lane == 0) mbar_arrive(&sm.freed[buf]);
      if (last_c) {
        const int bg = it_c / splits, split = it_c - bg * splits;
        const int b = bg / Hkv, g = bg - b * Hkv;
        float* st_o = reinterpret_cast<float*>(sm.ring[slot]);  // [warps][G][128]
        float* st_m = st_o + kPkWarps * G * kD;                  // [warps][G]
        float* st_l = st_m + kPkWarps * G;
        float ls = lsum;
        ls += __shfl_xor_sync(0xffffffffu, ls, 1);
        ls += __shfl_xor_sync(0xffffffffu, ls, 2);
        named_sync(2, kPkThreads);  // every consumer warp is done reading the slot
        {
          const int h0 = qc2, h1 = qc2 + 1;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            if (h0 < G) {
              st_o[(warp * G + h0) * kD + 16 * i + qr] = oT[i][0];
              st_o[(warp * G + h0) * kD + 16 * i + qr + 8] = oT[i][2];
            }
            if (h1 < G) {
              st_o[(warp * G + h1) * kD + 16 * i + qr] = oT[i][1];
              st_o[(warp * G + h1) * kD + 16 * i + qr + 8] = oT[i][3];
            }
          }
        }
        if (qr < G && (lane & 3) == 0) {
          st_m[warp * G + qr] = m;
          st_l[warp * G + qr] = ls;
        }
        named_sync(2, kPkThreads);
        const int d = tid;  // 128 consumer threads == 128 dims
        for (int j = 0; j < G; ++j) {
          float M = -INFINITY;
#pragma unroll
          for (int w = 0; w < kPkWarps; ++w) M = fmaxf(M, st_m[w * G + j]);
          float L = 0.f, O = 0.f;
          if (M != -INFINITY) {
#pragma unroll
            for (int w = 0; w < kPkWarps; ++w) {
              const float mw = st_m[w * G + j];
              if (mw != -INFINITY) {
                const float c = exp2f(mw - M);
                L = fmaf(st_l[w * G + j], c, L);
                O = fmaf(st_o[(w * G + j) * kD + d], c, O);
              }
            }
          }
          float* dst = part + (((size_t)b * Hq + g * G + j) * splits + split) * kPartStride;
          const uint64_t pol = l2_policy_evict_last();  // re-read by merge_parts_kernel
          st_keep_f32(dst + 2 + d, O, pol);
          if (d == 0) {
            st_keep_f32(dst, M, pol);
            st_keep_f32(dst + 1, L, pol);
          }
        }
        named_sync(2, kPkThreads);  // scratch read by all before the slot is released
        if (lane == 0) mbar_arrive(&sm.empty[slot]);
      }
    }
  }
  pdl_launch_dependents();
}

template <int G>
cudaError_t launch_pk_t(const Geo& g, const sd_paged_kv& kv, const void* q, const uint32_t* fbm, int ldw,
                        float scale, float* part, void* out, float* lse, int* counters, cudaStream_t st,
                        cudaEvent_t ev_attend) {
  const int splits = (g.max_seq_len + kPkItemTok - 1) / kPkItemTok;
  const int n_items = splits * g.B * g.Hkv;
  const size_t smem = sizeof(WsSmem<G>);
  static_assert(sizeof(float) * kPkWarps * G * (kD + 2) <= kPkStageBytes, "epilogue scratch fits a ring slot");
  auto kern = attend_union_ws_kernel<G>;
  cudaError_t e = ensure_dyn_smem(reinterpret_cast<const void*>(kern), smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(std::min(n_items, 2 * g.sms));
  cfg.blockDim = dim3(kWsThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, kern, reinterpret_cast<const uint16_t*>(q),
                         reinterpret_cast<const char*>(kv.k_pages), reinterpret_cast<const char*>(kv.v_pages),
                         kv.page_table, kv.seq_lens, g.max_seq_len, g.max_pages, g.Hkv, fbm, ldw, scale * kLog2e, part, splits,
                         n_items, counters + g.B * g.Hkv);
  if (e != cudaSuccess) return e;
  if (ev_attend) cudaEventRecord(ev_attend, st);
  return launch_merge_parts_pdl(part, g.B * g.Hq, splits, out, g.out_dtype, lse, st);
}

// Index lists -> selection bitmap rows (sd_sparse_gather_attend's union path).
// One CTA per q-row; rows up to kI2bWords * 32 tokens are assembled in shared
// memory and stored word by word, longer rows are zeroed and set in place.
constexpr int kI2bNT = 256;
constexpr int kI2bWords = 8192;
__global__ void __launch_bounds__(kI2bNT) idx_to_bits_kernel(const int* __restrict__ idx,
                                                             const int* __restrict__ counts, int k_max,
                                                             const int* __restrict__ seq_lens, int max_len, int Hq,
                                                             uint32_t* __restrict__ fbm, int ldw, int* __restrict__ work,
                                                             int* __restrict__ err) {
  __shared__ uint32_t sw[kI2bWords];
  const int row = blockIdx.x, b = row / Hq, tid = threadIdx.x;
  if (row == 0 && tid == 0) *work = 0;
  const int N = seq_len_dev(seq_lens, b, max_len);  // -1 (out of range): every count is rejected
  int cnt = __ldg(counts + row);
  if (cnt < 1 || cnt > k_max || cnt > N) {
    if (tid == 0) set_error(err, cnt < 1 ? SD_DEVERR_EMPTY : SD_DEVERR_SEQLEN);
    cnt = max(0, min(cnt, min(k_max, max(N, 0))));
  }
  const int nw = (max(N, 0) + 31) >> 5;
  uint32_t* fr = fbm + (size_t)row * ldw;
  const bool in_smem = nw <= kI2bWords;
  uint32_t* tw = in_smem ? sw : fr;
  for (int w = tid; w < nw; w += kI2bNT) tw[w] = 0u;
  __syncthreads();
  const int* ip = idx + (size_t)row * k_max;
  for (int e = tid; e < cnt; e += kI2bNT) {
    const int t = __ldg(ip + e);
    bool ok = t >= 0 && t < N;
    if (ok && e > 0 && __ldg(ip + e - 1) >= t) {
      ok = false;
      set_error(err, SD_DEVERR_INDEX_ORDER);
    } else if (!ok) {
      set_error(err, SD_DEVERR_INDEX_RANGE);
    }
    if (ok) atomicOr(tw + (t >> 5), 1u << (t & 31));
  }
  if (in_smem) {
    __syncthreads();
    for (int w = tid; w < nw; w += kI2bNT) fr[w] = sw[w];
  }
}

}  // namespace

cudaError_t launch_idx_to_bits(const Geo& g, const int* seq_lens, const int* idx, const int* counts, int k_max,
                               uint32_t* fbm, int ldw, int* work, int* err, cudaStream_t st) {
  idx_to_bits_kernel<<<g.B * g.Hq, kI2bNT, 0, st>>>(idx, counts, k_max, seq_lens, g.max_seq_len, g.Hq, fbm, ldw,
                                                    work, err);
  return cudaGetLastError();
}

cudaError_t launch_attend_union_pk(const Geo& g, const sd_paged_kv& kv, const void* q, const uint32_t* fbm, int ldw,
                                   float scale, float* part, void* out, float* lse, int* counters, cudaStream_t st,
                                   cudaEvent_t ev_attend) {
  switch (g.G) {
    case 1: return launch_pk_t<1>(g, kv, q, fbm, ldw, scale, part, out, lse, counters, st, ev_attend);
    case 2: return launch_pk_t<2>(g, kv, q, fbm, ldw, scale, part, out, lse, counters, st, ev_attend);
    case 4: return launch_pk_t<4>(g, kv, q, fbm, ldw, scale, part, out, lse, counters, st, ev_attend);
    case 8: return launch_pk_t<8>(g, kv, q, fbm, ldw, scale, part, out, lse, counters, st, ev_attend);
  }
  return cudaErrorInvalidValue;
}

}  // namespace sd

#ifdef SD_ATTEND_TRACE
extern "C" int sd_debug_attend_trace(unsigned long long* host, int n_ctas) {
  return (int)cudaMemcpyFromSymbol(host, sd::g_attend_trace, sizeof(unsigned long long) * 4 * n_ctas);
}
#endif
