// tools/micro/atoms.cu -- shared-memory atomic-min throughput on B200 (
// tuning aid, not product).  The build (K2) does M = 3 `red.shared.min.u32` per weight
// on bank-private keys; whether those atomics or HBM bound the build depends on this rate.
//   red-private : lane L always hits bank L (random row within its private column) -- K2's layout
//   red-random  : random word in a 32 K-word table (bank conflicts as they fall)
//   red-same    : all 32 lanes on one word (fully serialised)
//   atom-private: atom.shared.min (returns the old value) on the private layout
//   lds-private : plain ld.shared on the same addresses (the LSU floor, one wavefront per warp op)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o atoms tools/micro/atoms.cu && ./atoms
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void __launch_bounds__(512, 1) kern(uint32_t* out, int iters) {
  extern __shared__ uint32_t sm[];
  const int words = 32768;
  for (int i = threadIdx.x; i < words; i += blockDim.x) sm[i] = 0xFFFFFFFFu;
  __syncthreads();
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(sm);
  const int lane = threadIdx.x & 31;
  // 8 random addresses per thread, precomputed: the timed loop issues only the shared-memory ops
  uint32_t ad[8];
  uint32_t h = threadIdx.x * 0x9E3779B9u + blockIdx.x * 0x85EBCA6Bu;
  for (int k = 0; k < 8; ++k) {
    h = h * 1664525u + 1013904223u;
    if (MODE == 0 || MODE == 3 || MODE == 4) ad[k] = base + ((h >> 22) << 7) + 4u * lane;  // 1024 rows x 32 banks
    else if (MODE == 1) ad[k] = base + ((h >> 17) << 2);
    else ad[k] = base;
  }
  uint32_t acc = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const uint32_t addr = ad[k], v = (uint32_t)it ^ h;
      if (MODE == 3) {
        uint32_t old;
        asm volatile("atom.shared.min.u32 %0, [%1], %2;" : "=r"(old) : "r"(addr), "r"(v) : "memory");
        acc += old;
      } else if (MODE == 4) {
        uint32_t w;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(w) : "r"(addr) : "memory");
        acc ^= w;
      } else {
        asm volatile("red.shared.min.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = sm[lane] + acc;
  if (acc == 0x12345) out[blockIdx.x + 1] = acc;
}

template <int MODE>
void run(const char* name) {
  const size_t smem = 32768 * 4;
  cudaFuncSetAttribute(kern<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  uint32_t* out;
  cudaMalloc(&out, 4096 * 4);
  const int iters = MODE == 2 ? 200 : 4000;
  kern<MODE><<<148, 512, smem>>>(out, iters);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) kern<MODE><<<148, 512, smem>>>(out, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double ops = 5.0 * 148 * 512 * (double)iters * 8;  // lane-ops
  const double per_clk_sm = ops / (ms * 1e-3) / 148 / 1.965e9;
  printf("%-13s %8.1f G lane-ops/s  %6.2f lane-ops/clk/SM  (%.2f clk per warp op per SM) %s\n", name, ops / ms / 1e6,
         per_clk_sm, 32.0 / per_clk_sm, cudaGetErrorString(cudaGetLastError()));
  cudaFree(out);
}

int main() {
  run<0>("red-private");
  run<1>("red-random");
  run<2>("red-same");
  run<3>("atom-private");
  run<4>("lds-private");
  return 0;
}
