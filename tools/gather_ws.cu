// gather_ws.cu - producer / consumer variant of gather_ceiling.cu: per CTA, NP
// producer threads gather 256-B K/V rows (random pages, cfg3 union pattern)
// with 16-B cp.async into an NS-stage ring and signal each stage with
// cp.async.mbarrier.arrive.noinc; 128 consumer threads wait on the stage's
// mbarrier, touch it and release it.  Measures the HBM rate a warp-specialised
// gather-attend could reach (no compute).
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/gws tools/gather_ws.cu
//   /tmp/gws [ctas_per_sm] [stages] [producer threads: 128 | 256]
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <random>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  asm volatile(
      "{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W;\n}" ::"r"(su32(b)),
      "r"(ph)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void cp_arrive_noinc(uint64_t* b) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void cp16(uint32_t d, const void* s) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(s) : "memory");
}

template <int NS, int NP>
__global__ void __launch_bounds__(128 + NP) gather_ws(const char* kp, const char* vp, const uint32_t* rows, int nrows,
                                                      int rows_per_cta, unsigned long long* sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + NS * 32768);
  uint64_t* empty = full + NS;
  uint32_t* srow = reinterpret_cast<uint32_t*>(empty + NS);
  const int tid = threadIdx.x;
  const int r_begin = blockIdx.x * rows_per_cta, r_end = min(nrows, r_begin + rows_per_cta);
  const int nst = (r_end - r_begin + 63) / 64;
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(full + s, NP);
      mbar_init(empty + s, 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int r = r_begin + tid; r < r_end; r += blockDim.x) srow[r - r_begin] = rows[r];
  __syncthreads();
  if (tid >= 128) {  // producers
    const int p = tid - 128, ic = p & 15, ir0 = p >> 4;
    constexpr int RSTEP = NP / 16;
    for (int s = 0; s < nst; ++s) {
      const int slot = s % NS;
      if (s >= NS) mbar_wait(empty + slot, ((s / NS) - 1) & 1);
      unsigned char* st = sm + slot * 32768;
      for (int rr = ir0; rr < 64; rr += RSTEP) {
        const int r = r_begin + s * 64 + rr;
        if (r < r_end) {
          const size_t off = (size_t)srow[r - r_begin] * 256 + ic * 16;
          const uint32_t d = su32(st + rr * 256 + ic * 16);
          cp16(d, kp + off);
          cp16(d + 16384, vp + off);
        }
      }
      cp_arrive_noinc(full + slot);
    }
  } else {  // consumers
    unsigned long long acc = 0;
    for (int s = 0; s < nst; ++s) {
      const int slot = s % NS;
      mbar_wait(full + slot, (s / NS) & 1);
      acc += sm[slot * 32768 + tid * 4];
      __syncwarp();
      if ((tid & 31) == 0) mbar_arrive(empty + slot);
    }
    if (acc == 0x7fffffff) sink[0] = acc;
  }
}

int main(int argc, char** argv) {
  const int ctas_per_sm = argc > 1 ? atoi(argv[1]) : 2;
  const int stages = argc > 2 ? atoi(argv[2]) : 3;
  const int np = argc > 3 ? atoi(argv[3]) : 128;
  const int B = 16, Hkv = 8, N = 131072, PS = 16;
  const size_t pages = (size_t)B * N / PS;
  const size_t bytes = pages * PS * Hkv * 128 * 2;
  char *kp, *vp;
  cudaMalloc(&kp, bytes);
  cudaMalloc(&vp, bytes);
  cudaMemset(kp, 1, bytes);
  cudaMemset(vp, 1, bytes);
  std::mt19937_64 rng(1);
  std::vector<uint32_t> perm(pages);
  for (size_t i = 0; i < pages; ++i) perm[i] = (uint32_t)i;
  std::shuffle(perm.begin(), perm.end(), rng);
  std::vector<uint32_t> rows;
  const int per = 9616;
  for (int b = 0; b < B; ++b)
    for (int g = 0; g < Hkv; ++g) {
      std::vector<int> toks;
      std::uniform_int_distribution<int> U(0, N - 1);
      for (int t = 0; t < per; ++t) toks.push_back(U(rng));
      std::sort(toks.begin(), toks.end());
      toks.erase(std::unique(toks.begin(), toks.end()), toks.end());
      for (int t : toks) {
        const uint32_t page = perm[(size_t)b * (N / PS) + t / PS];
        rows.push_back((page * PS + t % PS) * Hkv + g);
      }
    }
  uint32_t* d_rows;
  cudaMalloc(&d_rows, rows.size() * 4);
  cudaMemcpy(d_rows, rows.data(), rows.size() * 4, cudaMemcpyHostToDevice);
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int nrows = (int)rows.size(), ctas = sms * ctas_per_sm;
  const int rpc = ((nrows + ctas - 1) / ctas + 63) / 64 * 64;
  const size_t smem = (size_t)stages * 32768 + 16 * stages + (size_t)rpc * 4;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 6; ++rep) {
    cudaEventRecord(e0);
#define L(S, P)                                                                                      \
  if (stages == S && np == P) {                                                                      \
    cudaFuncSetAttribute(gather_ws<S, P>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);    \
    gather_ws<S, P><<<ctas, 128 + P, smem>>>(kp, vp, d_rows, nrows, rpc, sink);                      \
  }
    L(2, 128) L(3, 128) L(4, 128) L(2, 256) L(3, 256) L(4, 256)
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep > 0) best = std::min(best, ms);
  }
  const double gb = (double)nrows * 512 / 1e9;
  printf("ws: producers %d stages %d ctas %d (%d/SM): %.1f MB, %.1f us, %.0f GB/s  [%s]\n", np, stages, ctas, ctas_per_sm,
         gb * 1e3, best * 1e3, gb / (best * 1e-3), cudaGetErrorString(cudaGetLastError()));
  return 0;
}
