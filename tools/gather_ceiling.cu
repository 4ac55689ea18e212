// gather_ceiling.cu - measures the HBM bandwidth a B200 sustains for gathers of
// 256-B K/V rows at random (page, slot) positions of a paged bf16 cache, the
// access pattern of the union gather-attend at N = 128K, S = 50 (cfg3).  No
// compute: every CTA streams its rows with 16-B cp.async into a shared-memory
// ring of `stages` x 32 KB (64 rows of K + 64 of V) and discards them.
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/gc tools/gather_ceiling.cu
//   /tmp/gc [ctas_per_sm] [stages] [pattern: 0 random, 1 sorted random, 2 sequential]
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <stdint.h>
#include <algorithm>
#include <vector>
#include <random>

__device__ __forceinline__ void cp16(uint32_t d, const void* s) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(s) : "memory");
}
template <int STAGES>
__global__ void __launch_bounds__(512) gather(const char* kp, const char* vp, const uint32_t* rows, int nrows,
                                              int rows_per_cta, unsigned long long* sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  const int tid = threadIdx.x, ic = tid & 15, ir0 = tid >> 4;
  const int rstep = blockDim.x >> 4;  // rows per pass of the CTA
  const int r_begin = blockIdx.x * rows_per_cta, r_end = min(nrows, r_begin + rows_per_cta);
  const int nst = (r_end - r_begin + 63) / 64;
  // the CTA's row indices are staged in shared memory first (as the attend
  // kernels hold them), so the copy issue never waits on a global load
  uint32_t* srow = reinterpret_cast<uint32_t*>(sm + STAGES * 32768);
  for (int r = r_begin + tid; r < r_end; r += blockDim.x) srow[r - r_begin] = rows[r];
  __syncthreads();
  auto issue = [&](int s) {
    if (s < nst) {
      unsigned char* st = sm + (s % STAGES) * 32768;
      for (int rr = ir0; rr < 64; rr += rstep) {
        const int r = r_begin + s * 64 + rr;
        if (r < r_end) {
          const size_t off = (size_t)srow[r - r_begin] * 256 + ic * 16;
          const uint32_t d = (uint32_t)__cvta_generic_to_shared(st + rr * 256 + ic * 16);
          cp16(d, kp + off);
          cp16(d + 16384, vp + off);
        }
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  for (int s = 0; s < STAGES - 1; ++s) issue(s);
  unsigned long long acc = 0;
  for (int s = 0; s < nst; ++s) {
    issue(s + STAGES - 1);
    asm volatile("cp.async.wait_group %0;" ::"n"(STAGES - 1) : "memory");
    __syncthreads();
    acc += sm[(s % STAGES) * 32768 + (tid & 127) * 4];
    __syncthreads();
  }
  if (acc == 0x7fffffff) sink[0] = acc;
}

int main(int argc, char** argv) {
  const int ctas_per_sm = argc > 1 ? atoi(argv[1]) : 2;
  const int stages = argc > 2 ? atoi(argv[2]) : 3;
  const int pattern = argc > 3 ? atoi(argv[3]) : 0;
  const int nt = argc > 4 ? atoi(argv[4]) : 128;
  const int B = 16, Hkv = 8, N = 131072, PS = 16;
  const size_t pages = (size_t)B * N / PS;
  const size_t bytes = pages * PS * Hkv * 128 * 2;
  char *kp, *vp;
  cudaMalloc(&kp, bytes);
  cudaMalloc(&vp, bytes);
  cudaMemset(kp, 1, bytes);
  cudaMemset(vp, 1, bytes);
  // rows: per (b, g), ~9600 distinct random tokens of a 131072-token sequence
  // with randomly permuted pages (the cfg3 union size), ascending per group
  std::mt19937_64 rng(1);
  std::vector<uint32_t> perm(pages);
  for (size_t i = 0; i < pages; ++i) perm[i] = (uint32_t)i;
  std::shuffle(perm.begin(), perm.end(), rng);
  std::vector<uint32_t> rows;
  const int per = 9616;
  for (int b = 0; b < B; ++b)
    for (int g = 0; g < Hkv; ++g) {
      std::vector<int> toks;
      if (pattern == 2) {
        for (int t = 0; t < per; ++t) toks.push_back(t);
      } else {
        std::uniform_int_distribution<int> U(0, N - 1);
        for (int t = 0; t < per; ++t) toks.push_back(U(rng));
        std::sort(toks.begin(), toks.end());
        toks.erase(std::unique(toks.begin(), toks.end()), toks.end());
      }
      for (int t : toks) {
        const uint32_t page = perm[(size_t)b * (N / PS) + t / PS];
        rows.push_back((page * PS + t % PS) * Hkv + g);
      }
    }
  if (pattern == 0) std::shuffle(rows.begin(), rows.end(), rng);
  uint32_t* d_rows;
  cudaMalloc(&d_rows, rows.size() * 4);
  cudaMemcpy(d_rows, rows.data(), rows.size() * 4, cudaMemcpyHostToDevice);
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int nrows = (int)rows.size();
  auto run = [&](int ctas) {
    const int rpc = ((nrows + ctas - 1) / ctas + 63) / 64 * 64;
    const size_t smem = (size_t)stages * 32768 + (size_t)rpc * 4;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 6; ++rep) {
      cudaEventRecord(e0);
      switch (stages) {
        case 2: cudaFuncSetAttribute(gather<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                gather<2><<<ctas, nt, smem>>>(kp, vp, d_rows, nrows, rpc, sink); break;
        case 3: cudaFuncSetAttribute(gather<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                gather<3><<<ctas, nt, smem>>>(kp, vp, d_rows, nrows, rpc, sink); break;
        case 4: cudaFuncSetAttribute(gather<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                gather<4><<<ctas, nt, smem>>>(kp, vp, d_rows, nrows, rpc, sink); break;
        case 6: cudaFuncSetAttribute(gather<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                gather<6><<<ctas, nt, smem>>>(kp, vp, d_rows, nrows, rpc, sink); break;
      }
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep > 0) best = std::min(best, ms);
    }
    const double gb = (double)nrows * 512 / 1e9;
    printf("threads %d pattern %d stages %d ctas %d (%d/SM): rows %d, %.1f MB, %.1f us, %.0f GB/s\n", nt, pattern, stages, ctas,
           ctas / sms, nrows, gb * 1e3, best * 1e3, gb / (best * 1e-3));
  };
  run(sms * ctas_per_sm);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) printf("error: %s\n", cudaGetErrorString(err));
  return 0;
}
