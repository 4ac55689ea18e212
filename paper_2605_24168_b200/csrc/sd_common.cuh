// sd_common.cuh - device primitives shared by the sdattn kernels (sm_100a).
//
// Layout contract (include/sdattn.h): head_dim D = 128, page_size = 16,
// K/V pages [num_pages][16][Hkv][128] (NHD), sketch pages
// [num_pages][Hkv][16][C] bf16.  One K or V row of one KV head is 256 B (bf16)
// or 512 B (fp32) contiguous; a half-warp (16 lanes) covers it with one 16-B
// (bf16) or two 16-B (fp32) vector loads per lane.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "sdattn.h"

namespace sd {

constexpr int kD = 128;         // head_dim
constexpr int kPS = 16;         // page size
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

// ---------------------------------------------------------------- error word
__device__ __forceinline__ void set_error(int* err, int code) {
  if (err) atomicCAS(err, 0, code);
}

// ---------------------------------------------------------------- intake (A1)
// N_b read against the HOST bound max_seq_len that sized the grids and the
// workspace (sdattn.h: 1 <= N_b <= max_seq_len).  A length outside [0, max_len]
// reads as -1: every kernel treats the row as empty (nothing is read or written
// past the workspace rows) and the kernels that own the row's result report
// SD_DEVERR_SEQLEN.  0 is returned as 0 (an empty local shard is legal for the
// sequence-shard entries; the other entries reject it as SEQLEN).
__device__ __forceinline__ int seq_len_dev(const int* __restrict__ seq_lens, int b, int max_len) {
  const int n = __ldg(seq_lens + b);
  return (n >= 0 && n <= max_len) ? n : -1;
}

// ---------------------------------------------------------------- budget (A1)
// k_b = max(1, ceil(N / S)) in double precision, or k_fixed.
__device__ __forceinline__ int budget_k_dev(int N, double S, int k_fixed) {
  if (k_fixed > 0) return k_fixed;
  double q = (double)N / S;
  double c = ceil(q);
  int k = c < 1.0 ? 1 : (c > (double)N ? N : (int)c);
  return k;
}

// NEXT-1 (Sink + Local + heavy): with n_sink, n_local or
// heavy_fraction non-zero the row keeps the sinks [0, lo) and the locals
// [hi, N) (lo = min(n_sink, N), hi = max(lo, N - min(n_local, N))) plus the
// top-kh tokens of the middle [lo, hi): kh = min(k_fixed, mid) if k_fixed > 0,
// else min(mid, floor(heavy_fraction * mid + 1/2)) (round half up).
// Implemented everywhere as "sink / local tokens score +inf" and a total
// k = lo + (N - hi) + kh, so the selection stays a plain top-k.
struct BudgetDev {
  double S;
  int k_fixed, n_sink, n_local;
  double heavy_fraction;
  // sequence shard: k_b from the sequence's GLOBAL length
  // kfrom[b] (<= max_from), at most the local N_b; null: from the local N_b
  const int* kfrom = nullptr;
  int max_from = 0;
};
struct RowBudget {
  int lo, hi, k;  // middle region [lo, hi), total selected k (0 allowed in NEXT-1 mode)
};
__device__ __forceinline__ bool budget_regions(const BudgetDev& b) {
  return b.n_sink != 0 || b.n_local != 0 || b.heavy_fraction != 0.0;
}
__device__ __forceinline__ RowBudget row_budget(int N, const BudgetDev& b) {
  RowBudget r;
  if (!budget_regions(b)) {
    r.lo = 0;
    r.hi = N;
    r.k = budget_k_dev(N, b.S, b.k_fixed);
    return r;
  }
  r.lo = min(b.n_sink, N);
  r.hi = max(r.lo, N - min(b.n_local, N));
  const int mid = r.hi - r.lo;
  int kh;
  if (b.k_fixed > 0) kh = min(b.k_fixed, mid);
  else kh = min(mid, (int)floor(b.heavy_fraction * (double)mid + 0.5));
  r.k = r.lo + (N - r.hi) + kh;
  return r;
}

// k_b of a sequence shard: from the global length, at most the local N (-1: invalid global length).
__device__ __forceinline__ int shard_row_k(const BudgetDev& b, int bi, int N) {
  const int NG = seq_len_dev(b.kfrom, bi, b.max_from);
  return NG >= 1 ? min(budget_k_dev(NG, b.S, b.k_fixed), max(N, 0)) : -1;
}

// ---------------------------------------------------------------- radix keys
// Order-preserving map fp32 -> uint32 (larger score -> larger key).  -0.0 is
// canonicalised to +0.0 so that equal scores give equal keys (ties then go to
// the lower index).  Scores are finite by precondition.
__device__ __forceinline__ uint32_t score_key(float f) {
  uint32_t u = __float_as_uint(f);
  if (u == 0x80000000u) u = 0u;
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float key_score(uint32_t k) {
  uint32_t u = (k & 0x80000000u) ? (k & 0x7fffffffu) : ~k;
  return __uint_as_float(u);
}

// ---------------------------------------------------------------- loads
__device__ __forceinline__ uint4 ldg_nc_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ uint4 ldg_v4(const void* p) {
  return __ldg(reinterpret_cast<const uint4*>(p));
}

__device__ __forceinline__ float bf_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf_hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }

__device__ __forceinline__ void unpack_bf16x8(const uint4& v, float* f) {
  f[0] = bf_lo(v.x); f[1] = bf_hi(v.x);
  f[2] = bf_lo(v.y); f[3] = bf_hi(v.y);
  f[4] = bf_lo(v.z); f[5] = bf_hi(v.z);
  f[6] = bf_lo(v.w); f[7] = bf_hi(v.w);
}

// Element type traits: 8 consecutive elements of a row as raw vector(s).
struct KvBF16 {
  static constexpr int kBytes = 2;
  struct Raw { uint4 a; };
  __device__ __forceinline__ static Raw load(const void* base, size_t elem) {
    Raw r; r.a = ldg_nc_v4(reinterpret_cast<const char*>(base) + elem * 2); return r;
  }
  __device__ __forceinline__ static void unpack(const Raw& r, float* f) { unpack_bf16x8(r.a, f); }
};
struct KvF32 {
  static constexpr int kBytes = 4;
  struct Raw { uint4 a, b; };
  __device__ __forceinline__ static Raw load(const void* base, size_t elem) {
    const char* p = reinterpret_cast<const char*>(base) + elem * 4;
    Raw r; r.a = ldg_nc_v4(p); r.b = ldg_nc_v4(p + 16); return r;
  }
  __device__ __forceinline__ static void unpack(const Raw& r, float* f) {
    f[0] = __uint_as_float(r.a.x); f[1] = __uint_as_float(r.a.y);
    f[2] = __uint_as_float(r.a.z); f[3] = __uint_as_float(r.a.w);
    f[4] = __uint_as_float(r.b.x); f[5] = __uint_as_float(r.b.y);
    f[6] = __uint_as_float(r.b.z); f[7] = __uint_as_float(r.b.w);
  }
};

// q row chunk (8 elements at d0) as fp32, q stored in the KV dtype.
template <class KV>
__device__ __forceinline__ void load_q8(const void* q, size_t elem, float* f) {
  typename KV::Raw r;
  if (KV::kBytes == 2) {
    r.a = ldg_v4(reinterpret_cast<const char*>(q) + elem * 2);
  } else {
    const char* p = reinterpret_cast<const char*>(q) + elem * 4;
    reinterpret_cast<uint4*>(&r)[0] = ldg_v4(p);
    reinterpret_cast<uint4*>(&r)[1] = ldg_v4(p + 16);
  }
  KV::unpack(r, f);
}

// Element offset of row (page, slot, kv head g) in a [P][16][Hkv][128] pool.
__device__ __forceinline__ size_t kv_row_elem(int page, int slot, int g, int Hkv) {
  return ((size_t)(page * kPS + slot) * Hkv + g) * kD;
}

// ---------------------------------------------------------------- output store
__device__ __forceinline__ void store_out(void* out, int out_dtype, size_t i, float v) {
  if (out_dtype == SD_F32) {
    reinterpret_cast<float*>(out)[i] = v;
  } else {
    uint32_t u = __float_as_uint(v);
    // round to nearest even (finite inputs)
    u += 0x7fffu + ((u >> 16) & 1u);
    reinterpret_cast<uint16_t*>(out)[i] = (uint16_t)(u >> 16);
  }
}

// ---------------------------------------------------------------- mbarrier + bulk copy (TMA engine)
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "SD_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra SD_WAIT;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// 1-D bulk async copy global -> shared (cp.async.bulk, executed by the TMA
// unit); completion is signalled as `bytes` transactions on `bar`.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// ---------------------------------------------------------------- L2 cache policy
// Evict-last stores for small results a later kernel of the step re-reads
// (band entries, selection words, split partials) while ~900 MB of sketch and
// K/V rows stream through L2.
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void st_keep_u32(uint32_t* p, uint32_t v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.u32 [%0], %1, %2;" ::"l"(p), "r"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_keep_f32(float* p, float v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(p), "f"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_keep_f2(float2* p, float2 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v2.f32 [%0], {%1, %2}, %3;" ::"l"(p), "f"(v.x), "f"(v.y), "l"(pol) : "memory");
}

// Programmatic dependent launch (PDL): let the next kernel in the stream start
// its prologue early / wait for the previous kernel's memory to be visible.
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// ---------------------------------------------------------------- reductions
__device__ __forceinline__ float half_warp_sum(float v) {
  v += __shfl_xor_sync(0xffffffffu, v, 8);
  v += __shfl_xor_sync(0xffffffffu, v, 4);
  v += __shfl_xor_sync(0xffffffffu, v, 2);
  v += __shfl_xor_sync(0xffffffffu, v, 1);
  return v;
}

}  // namespace sd
