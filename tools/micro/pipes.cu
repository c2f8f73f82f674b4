// Throughput of single integer/float ops on one SM (tuning aid): 8 independent chains per thread,
// 1024 threads per CTA, one CTA per SM; prints warp-instructions per clock per SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int OP>
__global__ void k(uint32_t* out, uint32_t a, uint32_t b, int iters) {
  uint32_t r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = threadIdx.x * (j + 3) + a;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (OP == 0) r[j] = r[j] * b + a;                          // IMAD
      if (OP == 1) r[j] = __umulhi(r[j], b) + a;                // IMAD.HI
      if (OP == 2) r[j] = (r[j] ^ b) + (r[j] >> 3);              // alu (LOP3 + LEA.HI / IADD)
      if (OP == 3) r[j] = __float_as_uint(__fmaf_rn(__uint_as_float(r[j]), 1.0001f, 0.5f));  // FFMA
      if (OP == 4) r[j] = __funnelshift_l(r[j], r[j], 7);        // SHF
      if (OP == 5) { uint64_t w = (uint64_t)r[j] * b; r[j] = (uint32_t)(w >> 32) ^ (uint32_t)w; }  // IMAD.WIDE
      if (OP == 6) r[j] = (r[j] * b) ^ __umulhi(r[j], a);        // IMAD + IMAD.HI mix
    }
  }
  long long t1 = clock64();
  uint32_t s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s ^= r[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) out[gridDim.x * blockDim.x + blockIdx.x] = (uint32_t)(t1 - t0);
}

template <int OP>
void run(const char* name, int ops_per_j) {
  const int T = 1024, G = 148, iters = 4096;
  uint32_t* d;
  cudaMalloc(&d, (G * T + G) * 4);
  k<OP><<<G, T>>>(d, 12345, 0x9E3779B1u, 16);
  k<OP><<<G, T>>>(d, 12345, 0x9E3779B1u, iters);
  cudaDeviceSynchronize();
  uint32_t cyc;
  cudaMemcpy(&cyc, d + G * T, 4, cudaMemcpyDeviceToHost);
  double warp_instr = (double)T / 32 * iters * 8 * ops_per_j;
  printf("%-10s %.3f warp-instr/clk/SM (%.2f clk per warp-instr per SMSP)\n", name, warp_instr / cyc,
         4.0 / (warp_instr / cyc));
  cudaFree(d);
}

int main() {
  run<0>("IMAD", 1);
  run<1>("IMAD.HI", 2);  // hi + add (add may fold into the IMAD.HI addend)
  run<2>("ALU(2)", 2);
  run<3>("FFMA", 1);
  run<4>("SHF", 1);
  run<5>("WIDE+LOP", 2);
  run<6>("IMAD,HI,LOP", 3);
  return 0;
}
