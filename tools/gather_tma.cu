// gather_tma.cu - TMA tile::gather4 variant of gather_ws.cu: the cfg3 union
// row pattern (random pages, 256-B K and V rows) gathered by one producer warp
// with cp.async.bulk.tensor.2d.tile::gather4 (4 rows per instruction) over 2-D
// tensor maps of the K / V pools viewed as [pages * 16 * Hkv rows][128] bf16,
// completion through mbarrier complete_tx; 4 consumer warps wait on the stage,
// touch it and release it.  Also checks the 128-B swizzle placement the attend
// relies on: row r, 16-B chunk c of a 64-row stage lands at
//   (c >> 3) * 8192 + r * 128 + (((c & 7) ^ (r & 7)) << 4)
// for the swizzled (2 half-boxes of 64 columns) layout.
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/gtma tools/gather_tma.cu -lcuda
//   /tmp/gtma [ctas_per_sm] [stages] [issuing lanes] [l2 promotion 0..3] [swizzle: 1 | 0 (box 128, no swizzle)]
#include <cuda.h>
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
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void gather4(uint32_t dst, const CUtensorMap* map, uint64_t* bar, int col, int r0, int r1,
                                        int r2, int r3) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
      "%5, %6}], [%7];" ::"r"(dst),
      "l"(map), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(su32(bar))
      : "memory");
}

template <int NS, bool SWZ>
__global__ void __launch_bounds__(160) gather_tma(const __grid_constant__ CUtensorMap kmap,
                                                  const __grid_constant__ CUtensorMap vmap, const uint32_t* rows,
                                                  int nrows, int rows_per_cta, int lanes, unsigned long long* sink,
                                                  int* bad) {
  extern __shared__ __align__(1024) unsigned char smraw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~(uintptr_t)1023);
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + NS * 32768);
  uint64_t* empty = full + NS;
  uint32_t* srow = reinterpret_cast<uint32_t*>(empty + NS);
  const int tid = threadIdx.x, lane = tid & 31;
  const int r_begin = blockIdx.x * rows_per_cta, r_end = min(nrows, r_begin + rows_per_cta);
  const int nst = (r_end - r_begin + 63) / 64;
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int r = r_begin + tid; r < r_end; r += blockDim.x) srow[r - r_begin] = rows[r];
  __syncthreads();
  if (tid >= 128) {  // producer warp
    for (int s = 0; s < nst; ++s) {
      const int slot = s % NS;
      if (s >= NS) mbar_wait(empty + slot, ((s / NS) - 1) & 1);
      const uint32_t st = su32(sm + slot * 32768);
      const int R0 = r_begin + s * 64, nr = min(64, r_end - R0);
      const int ng = (nr + 3) >> 2;                      // row groups of 4
      const int nops = SWZ ? ng * 4 : ng * 2;            // K/V x halves
      if (lane == 0) mbar_expect_tx(full + slot, (uint32_t)nops * 512u * (SWZ ? 1u : 2u));
      __syncwarp();
      for (int op = lane; op < nops && lane < lanes; op += lanes) {
        const int gi = SWZ ? (op >> 2) : (op >> 1);
        const int kv = SWZ ? ((op >> 1) & 1) : (op & 1);
        const int half = SWZ ? (op & 1) : 0;
        int r[4];
        for (int i = 0; i < 4; ++i) {
          const int rr = min(4 * gi + i, nr - 1);  // a ragged group repeats the last row
          r[i] = (int)srow[R0 - r_begin + rr];
        }
        const uint32_t dst = SWZ ? st + kv * 16384 + half * 8192 + gi * 512 : st + kv * 16384 + gi * 1024;
        gather4(dst, kv ? &vmap : &kmap, full + slot, half * 64, r[0], r[1], r[2], r[3]);
      }
    }
  } else {  // consumers: check the placement of the K rows' first words, touch the stage
    unsigned long long acc = 0;
    const int w = tid >> 5;
    for (int s = 0; s < nst; ++s) {
      const int slot = s % NS;
      mbar_wait(full + slot, (s / NS) & 1);
      const int R0 = r_begin + s * 64, nr = min(64, r_end - R0);
      // 128 threads: row (tid >> 1), chunk 0 or 15
      const int r = tid >> 1, c = (tid & 1) ? 15 : 0;
      if (r < nr) {
        const uint32_t off = SWZ ? (uint32_t)((c >> 3) * 8192 + r * 128 + (((c & 7) ^ (r & 7)) << 4))
                                 : (uint32_t)(r * 256 + c * 16);
        const uint32_t v = *reinterpret_cast<const uint32_t*>(sm + slot * 32768 + off);
        // K element (row R, col 8c) holds (R * 16 + c) as a 32-bit word
        const uint32_t want = srow[R0 - r_begin + r] * 16u + (uint32_t)c;
        if (v != want) atomicAdd(bad, 1);
        acc += v;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + slot);
    }
    (void)w;
    if (acc == 0x7fffffffffffull) sink[0] = acc;
  }
}

__global__ void fill_pattern(uint32_t* p, size_t rows) {
  // each 256-B row R: 16-B chunk c's first word = R * 16 + c
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < rows * 16; i += (size_t)gridDim.x * blockDim.x)
    p[i * 4] = (uint32_t)i;
}

int main(int argc, char** argv) {
  const int ctas_per_sm = argc > 1 ? atoi(argv[1]) : 2;
  const int stages = argc > 2 ? atoi(argv[2]) : 3;
  const int lanes = argc > 3 ? atoi(argv[3]) : 1;
  const int promo = argc > 4 ? atoi(argv[4]) : 3;
  const int swz = argc > 5 ? atoi(argv[5]) : 1;
  const int B = 16, Hkv = 8, N = 131072, PS = 16;
  const size_t pages = (size_t)B * N / PS;
  const size_t nrow_pool = pages * PS * Hkv;
  const size_t bytes = nrow_pool * 256;
  char *kp, *vp;
  cudaMalloc(&kp, bytes);
  cudaMalloc(&vp, bytes);
  fill_pattern<<<4096, 256>>>(reinterpret_cast<uint32_t*>(kp), nrow_pool);
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
  int* bad;
  cudaMalloc(&sink, 8);
  cudaMalloc(&bad, 4);
  cudaMemset(bad, 0, 4);

  CUtensorMap km, vm;
  const cuuint64_t gdim[2] = {128, (cuuint64_t)nrow_pool};
  const cuuint64_t gstr[1] = {256};
  const cuuint32_t box[2] = {swz ? 64u : 128u, 1u};
  const cuuint32_t es[2] = {1, 1};
  const CUtensorMapSwizzle sw = swz ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE;
  CUresult r1 = cuTensorMapEncodeTiled(&km, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, kp, gdim, gstr, box, es,
                                       CU_TENSOR_MAP_INTERLEAVE_NONE, sw, (CUtensorMapL2promotion)promo,
                                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  CUresult r2 = cuTensorMapEncodeTiled(&vm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, vp, gdim, gstr, box, es,
                                       CU_TENSOR_MAP_INTERLEAVE_NONE, sw, (CUtensorMapL2promotion)promo,
                                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r1 != CUDA_SUCCESS || r2 != CUDA_SUCCESS) {
    printf("cuTensorMapEncodeTiled failed: %d %d\n", (int)r1, (int)r2);
    return 1;
  }
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int nrows = (int)rows.size(), ctas = sms * ctas_per_sm;
  const int rpc = ((nrows + ctas - 1) / ctas + 63) / 64 * 64;
  const size_t smem = 1024 + (size_t)stages * 32768 + 16 * stages + (size_t)rpc * 4;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 6; ++rep) {
    cudaEventRecord(e0);
#define L(S, W)                                                                                                  \
  if (stages == S && swz == W) {                                                                                 \
    cudaFuncSetAttribute(gather_tma<S, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);              \
    gather_tma<S, W><<<ctas, 160, smem>>>(km, vm, d_rows, nrows, rpc, lanes, sink, bad);                         \
  }
    L(2, 1) L(3, 1) L(4, 1) L(6, 1) L(2, 0) L(3, 0) L(4, 0)
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep > 0) best = std::min(best, ms);
  }
  int h_bad = -1;
  cudaMemcpy(&h_bad, bad, 4, cudaMemcpyDeviceToHost);
  const double gb = (double)nrows * 512 / 1e9;
  printf("tma: swz %d lanes %d promo %d stages %d ctas %d (%d/SM): %.1f MB, %.1f us, %.0f GB/s, bad %d [%s]\n", swz,
         lanes, promo, stages, ctas, ctas_per_sm, gb * 1e3, best * 1e3, gb / (best * 1e-3), h_bad,
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
