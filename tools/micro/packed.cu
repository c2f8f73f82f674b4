// tools/micro/packed.cu -- round-2 ceiling of a PACKED decode inner loop (tuning aid, not product).
// Cells are 16-bit retrieve keys rho16 = rotl16(b, 1) ^ 1 of bf16 states; the UPL units of a lane
// share one hash (unit keys shared by groups of UPL units, L32), so one shared load of
// UPL * 2 bytes per sketch row fetches all of a lane's cells:
//   address_i(o) = FFMA.RZ(f_i(o), 512 N, c_i) * 512 + 16 L  (UPL = 8: LDS.128; UPL = 4: LDS.64)
// then VIMNMX3.U16x2 over the M = 3 rows (2 units per instruction), rotr16 of each half (-> bits of
// -w'), FHFMA.BF16 with -x.  Variants:
//   MODE 0: R_i(o) from a per-warp shared table (LDS.128 broadcast per row)
//   MODE 1: R_i(o) via SHFL from the lane that holds row r
//   MODE 2: MODE 0 with the >> 1 of the rotation as IMAD.HI (FMA pipe) instead of SHF (ALU pipe)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pk tools/micro/packed.cu && ./pk
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

template <int UPL>
struct Cells;
template <>
struct Cells<8> {
  uint32_t w[4];
};
template <>
struct Cells<4> {
  uint32_t w[2];
};

template <int UPL>
__device__ __forceinline__ void ldc(uint32_t a, Cells<UPL>& c) {
  if constexpr (UPL == 8)
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(c.w[0]), "=r"(c.w[1]), "=r"(c.w[2]), "=r"(c.w[3]) : "r"(a));
  else
    asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(c.w[0]), "=r"(c.w[1]) : "r"(a));
}
__device__ __forceinline__ uint32_t max3(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("max.u16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  asm("max.u16x2 %0, %1, %2;" : "=r"(d) : "r"(d), "r"(c));
  return d;
}
template <int MODE>
__device__ __forceinline__ uint32_t negw(uint32_t p) {  // rotr16 of both halves: bits of -w'
  uint32_t hi, d;
  if (MODE == 2) asm("mul.hi.u32 %0, %1, 0x80000000;" : "=r"(hi) : "r"(p));
  else hi = p >> 1;
  asm("lop3.b32 %0, %1, %2, 0x7FFF7FFF, 0xE4;" : "=r"(d) : "r"(hi), "r"(p << 15));
  return d;
}
__device__ __forceinline__ float fma_lo(uint32_t x, uint32_t w, float c) {
  float d;
  asm("{.reg .b16 wl, wh, xl, xh;\n\tmov.b32 {wl, wh}, %2;\n\tmov.b32 {xl, xh}, %1;\n\tfma.rn.f32.bf16 %0, xl, wl, %3;}"
      : "=f"(d) : "r"(x), "r"(w), "f"(c));
  return d;
}
__device__ __forceinline__ float fma_hi(uint32_t x, uint32_t w, float c) {
  float d;
  asm("{.reg .b16 wl, wh, xl, xh;\n\tmov.b32 {wl, wh}, %2;\n\tmov.b32 {xl, xh}, %1;\n\tfma.rn.f32.bf16 %0, xh, wh, %3;}"
      : "=f"(d) : "r"(x), "r"(w), "f"(c));
  return d;
}
template <int SUB>
__device__ __forceinline__ float transpose_reduce(float (&acc)[SUB], int lane) {
#pragma unroll
  for (int m = SUB / 2; m >= 1; m >>= 1) {
    const bool up = (lane & m) != 0;
#pragma unroll
    for (int i = 0; i < m; ++i) {
      const float send = up ? acc[i] : acc[i + m];
      const float keep = up ? acc[i + m] : acc[i];
      acc[i] = keep + __shfl_xor_sync(0xffffffffu, send, m);
    }
  }
  float t = acc[0];
#pragma unroll
  for (int m = SUB; m < 32; m <<= 1) t += __shfl_xor_sync(0xffffffffu, t, m);
  return t;
}

template <int UPL, int MODE, int SUB, int MAXREG>
__global__ void __launch_bounds__(512, 1) __maxnreg__(MAXREG) kern(float* out, int rows_per_warp, int N) {
  extern __shared__ __align__(1024) uint32_t sm[];
  constexpr int SL = 32 * UPL * 2;  // bytes per (i, k) slice
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int words = 3 * N * SL / 4;
  for (int i = threadIdx.x; i < words; i += blockDim.x) sm[i] = (i * 2654435761u) & 0x7FFF7FFFu;
  const uint32_t smb = ((uint32_t)__cvta_generic_to_shared(sm) + 1023u) & ~1023u;
  uint4* rt = reinterpret_cast<uint4*>(sm + words + 512) + warp * SUB;
  const uint32_t rtb = (uint32_t)__cvta_generic_to_shared(rt);
  __syncthreads();
  uint32_t fk[3], cb[3];
  const uint32_t K = 0x12345u + lane * 7777u;
  for (int i = 0; i < 3; ++i) {
    fk[i] = ((K * (2 * i + 7)) & 0x7FFFFFu) | 0x3F800000u;
    // result in [2^E, 2^(E+1)) with ulp SL: 2^E = SL * 2^23
    cb[i] = __float_as_uint((float)((double)SL * 8388608.0 + (double)(smb + (uint32_t)(i * N * SL)) - (double)SL * N));
  }
  const float NS = (float)(SL * N);
  const uint32_t LB = lane * (UPL * 2);
  uint32_t nx[UPL / 2];
  for (int v = 0; v < UPL / 2; ++v) nx[v] = 0xBF80BF80u + v;
  float tot = 0.f;
  for (int s = 0; s < rows_per_warp; s += SUB) {
    uint32_t rr0 = 0, rr1 = 0, rr2 = 0;
    const uint32_t o = (uint32_t)(blockIdx.x * 100000 + warp * 5000 + s + (lane & (SUB - 1)));
    auto fmix = [](uint32_t h) { h ^= h >> 16; h *= 0x85EBCA6Bu; h ^= h >> 13; h *= 0xC2B2AE35u; return h ^ (h >> 16); };
    if (MODE != 1) {
      __syncwarp();
      if (lane < SUB)
        asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(rtb + 16u * lane), "r"(fmix(o ^ 0x1111u) & 0x7FFFFFu),
                     "r"(fmix(o ^ 0x2222u) & 0x7FFFFFu), "r"(fmix(o ^ 0x3333u) & 0x7FFFFFu), "r"(0u)
                     : "memory");
      __syncwarp();
    } else {
      rr0 = fmix(o ^ 0x1111u) & 0x7FFFFFu;
      rr1 = fmix(o ^ 0x2222u) & 0x7FFFFFu;
      rr2 = fmix(o ^ 0x3333u) & 0x7FFFFFu;
    }
    float acc[SUB];
#pragma unroll
    for (int r = 0; r < SUB; ++r) {
      uint32_t R0, R1, R2;
      if (MODE != 1) {
        uint32_t pad;
        asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(R0), "=r"(R1), "=r"(R2), "=r"(pad) : "r"(rtb + 16u * r));
      } else {
        R0 = __shfl_sync(0xffffffffu, rr0, r);
        R1 = __shfl_sync(0xffffffffu, rr1, r);
        R2 = __shfl_sync(0xffffffffu, rr2, r);
      }
      const uint32_t Rv[3] = {R0, R1, R2};
      Cells<UPL> c[3];
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        const uint32_t bits = __float_as_uint(__fmaf_rz(__uint_as_float(Rv[i] ^ fk[i]), NS, __uint_as_float(cb[i])));
        ldc<UPL>(bits * (uint32_t)SL + LB, c[i]);
      }
      float a = 0.f;
#pragma unroll
      for (int p = 0; p < UPL / 2; ++p) {
        const uint32_t w = negw<MODE>(max3(c[0].w[p], c[1].w[p], c[2].w[p]));
        a = fma_lo(nx[p], w, a);
        a = fma_hi(nx[p], w, a);
      }
      acc[r] = a;
    }
    tot += transpose_reduce<SUB>(acc, lane);
  }
  if (tot == 1234.5f) out[blockIdx.x] = tot;
}

template <int UPL, int MODE, int SUB, int MAXREG>
void run(const char* name, int N) {
  constexpr int SL = 32 * UPL * 2;
  const size_t smem = (size_t)3 * N * SL + 2048 + 16 * 16 * 16 + 1024;
  auto k = kern<UPL, MODE, SUB, MAXREG>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  float* out;
  cudaMalloc(&out, 4096 * 4);
  const int rows = 4096;
  k<<<148, 512, smem>>>(out, rows, N);
  cudaError_t e0 = cudaDeviceSynchronize();
  if (e0 != cudaSuccess) {
    printf("%-14s UPL=%d: %s\n", name, UPL, cudaGetErrorString(e0));
    fflush(stdout);
    return;
  }
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) k<<<148, 512, smem>>>(out, rows, N);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double w = 5.0 * 148 * 16 * (double)rows * 32 * UPL;
  printf("%-14s UPL=%d SUB=%2d reg=%3d N=%3d  %8.1f Gweight/s  %6.2f weight/clk/SM @1965  %s\n", name, UPL, SUB, MAXREG, N,
         w / ms / 1e6, w / (ms * 1e-3) / 148 / 1.965e9, cudaGetErrorString(cudaGetLastError()));
  fflush(stdout);
  cudaFree(out);
}

int main() {
  for (int N : {85, 21}) {
    run<8, 0, 16, 112>("rtab-lds128", N);
    run<8, 1, 16, 112>("rtab-shfl", N);
    run<8, 2, 16, 112>("rtab-imadhi", N);
    run<8, 0, 16, 128>("rtab-lds128", N);
    run<8, 0, 8, 112>("rtab-lds128", N);
    run<4, 0, 16, 112>("u4-lds64", N);
    run<4, 2, 16, 112>("u4-imadhi", N);
  }
  return 0;
}
