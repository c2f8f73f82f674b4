// tools/micro/fhash.cu -- ceiling of the decode inner loop under the v2 hash contract (
// tuning aid, not product).  Per weight and sketch row: f = R_i ^ fkey (LOP3), q = FFMA.RZ(f, 4N, C)
// (bits 0x4C000000 + off + idx), address = q * 128 + lane base (IMAD), LDS; then VIMNMX3 + SHF + FFMA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fh tools/micro/fhash.cu && ./fh
// MODE 0: the v1 contract (IMAD + IMAD.HI + LEA per row); 1: v2 with 3 SHFL per row for R_i;
// 2: v2 with one LDS.128 broadcast of {R_0, R_1, R_2} per row (the product kernel's form);
// 3: as 2 with row 2's address from a LOP3 mask (C scaled by 128); 4: as 2 with LEA addresses.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t lds(uint32_t a) { uint32_t v; asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a)); return v; }
__device__ __forceinline__ uint32_t imad(uint32_t a, uint32_t b, uint32_t c) { uint32_t d; asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c)); return d; }

// MODE 0: baseline (current) ; 1: fhash SHFLx3, IMAD address ; 2: fhash LDS.128 broadcast, IMAD addr
// 3: fhash LDS.128, rows0,1 IMAD addr, row2 LOP3 mask addr ; 4: fhash LDS.128, LEA (shift+add) addr
template <int UPL, int MODE, int SUB>
__global__ void __launch_bounds__(512, 1) kern(const uint32_t* __restrict__ Rg, float* out, int rows_per_warp, int N) {
  extern __shared__ __align__(16) uint32_t sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int cells = UPL * 32 * 3 * (N + 1);
  for (int i = threadIdx.x; i < cells; i += blockDim.x) sm[i] = i * 2654435761u;
  uint4* rt = reinterpret_cast<uint4*>(sm + cells + 64) + warp * SUB;  // per-warp R table
  const uint32_t smb = (uint32_t)__cvta_generic_to_shared(sm);
  const uint32_t rtb = (uint32_t)__cvta_generic_to_shared(rt);
  __syncthreads();
  uint32_t K[UPL], Kf[UPL][3], C[UPL][3], B[UPL], B2[UPL][3];
  float Nf[UPL], Nf128[UPL];
  float nx[UPL];
  const uint32_t a0 = 0x9E3779B1u, a1 = 0x85EBCA77u, a2 = 0xC2B2AE3Du;
  for (int v = 0; v < UPL; ++v) {
    K[v] = 0x12345u * (v + 1) + lane;
    const uint32_t vb = (uint32_t)(v * 32 * 3 * (N + 1));
    B[v] = smb + 4u * (vb + lane);
    for (int i = 0; i < 3; ++i) {
      Kf[v][i] = ((K[v] * (i + 7)) & 0x7FFFFFu) | 0x3F800000u;
      C[v][i] = __float_as_uint((float)(33554432 - 4 * N + 4 * i * (N + 1)));
      B2[v][i] = smb + 4u * (vb + i * (N + 1) * 32);  // for the 128N form: C' = region byte offset
    }
    Nf[v] = (float)(4 * N);
    Nf128[v] = (float)(128 * N);
    nx[v] = 1.0f + v;
  }
  const uint32_t l4 = lane * 4u;
  float tot = 0.f;
  for (int s = 0; s < rows_per_warp; s += SUB) {
    const uint32_t Rl = Rg[(blockIdx.x * 512 + threadIdx.x + s) & 4095];
    uint32_t R0l = 0, R1l = 0, R2l = 0;
    if (MODE >= 1) {
      R0l = Rl & 0x7FFFFFu; R1l = (Rl * 0x2545F491u) >> 9; R2l = (Rl * 0x9E3779B9u) >> 9;
    }
    if (MODE >= 2) {
      if (lane < SUB) rt[lane] = make_uint4(R0l, R1l, R2l, 0);
      __syncwarp();
    }
    float acc[SUB];
#pragma unroll
    for (int r = 0; r < SUB; ++r) {
      uint32_t R0, R1, R2, Rv = 0;
      if (MODE == 0) Rv = __shfl_sync(0xffffffffu, Rl, r);
      else if (MODE == 1) {
        R0 = __shfl_sync(0xffffffffu, R0l, r); R1 = __shfl_sync(0xffffffffu, R1l, r); R2 = __shfl_sync(0xffffffffu, R2l, r);
      } else {
        uint4 q; asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(q.x), "=r"(q.y), "=r"(q.z), "=r"(q.w) : "r"(rtb + 16u * r));
        R0 = q.x; R1 = q.y; R2 = q.z;
      }
      float a = 0.f;
#pragma unroll
      for (int v = 0; v < UPL; ++v) {
        uint32_t m0, m1, m2;
        if (MODE == 0) {
          const uint32_t h = Rv ^ K[v];
          const uint32_t rb = smb + 4u * (uint32_t)(v * 32 * 3 * (N + 1) + lane);
          m0 = lds(rb + ((__umulhi(h * a0, N)) << 7));
          m1 = lds(rb + ((__umulhi(h * a1, N) + (N + 1)) << 7));
          m2 = lds(rb + ((__umulhi(h * a2, N) + 2 * (N + 1)) << 7));
        } else {
          const float f0 = __uint_as_float(R0 ^ Kf[v][0]);
          const float f1 = __uint_as_float(R1 ^ Kf[v][1]);
          const float f2 = __uint_as_float(R2 ^ Kf[v][2]);
          const uint32_t q0 = __float_as_uint(__fmaf_rz(f0, Nf[v], __uint_as_float(C[v][0])));
          const uint32_t q1 = __float_as_uint(__fmaf_rz(f1, Nf[v], __uint_as_float(C[v][1])));
          if (MODE == 3) {
            // 128N scaling at exponent 150 (ulp 1): mantissa = B2 + floor(128 k N / 2^23); mask to the row
            const uint32_t q2 = __float_as_uint(__fmaf_rz(f2, Nf128[v], __uint_as_float(0x4B000000u | (B2[v][2] - 128u * N))));
            m0 = lds(imad(q0, 128u, B[v]));
            m1 = lds(imad(q1, 128u, B[v]));
            m2 = lds((q2 & 0x7FFF80u) | l4);
          } else {
            const uint32_t q2 = __float_as_uint(__fmaf_rz(f2, Nf[v], __uint_as_float(C[v][2])));
            if (MODE == 4) {
              m0 = lds((q0 << 7) + B[v]); m1 = lds((q1 << 7) + B[v]); m2 = lds((q2 << 7) + B[v]);
            } else {
              m0 = lds(imad(q0, 128u, B[v])); m1 = lds(imad(q1, 128u, B[v])); m2 = lds(imad(q2, 128u, B[v]));
            }
          }
        }
        const uint32_t b = max(max(m0, m1), m2);
        a = fmaf(nx[v], __uint_as_float(__funnelshift_r(b, b, 1)), a);
      }
      acc[r] = a;
    }
#pragma unroll
    for (int r = 0; r < SUB; ++r) tot += acc[r];
    if (MODE >= 2) __syncwarp();
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = tot;
}

template <int UPL, int MODE, int SUB>
void run(const char* name) {
  const int N = 85;
  const size_t smem = (size_t)UPL * 32 * 3 * (N + 1) * 4 + 256 + 16 * 16 * SUB;
  cudaFuncSetAttribute(kern<UPL, MODE, SUB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int grid = 148;
  uint32_t* R; float* out;
  cudaMalloc(&R, 4096 * 4); cudaMemset(R, 7, 4096 * 4);
  cudaMalloc(&out, (size_t)grid * 512 * 4);
  const int rows = 16 * 128;
  kern<UPL, MODE, SUB><<<grid, 512, smem>>>(R, out, rows, N);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int it = 0; it < 5; ++it) kern<UPL, MODE, SUB><<<grid, 512, smem>>>(R, out, rows, N);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  cudaError_t e = cudaGetLastError();
  const double weights = 5.0 * grid * 512.0 * rows * UPL;
  printf("%-10s UPL=%d SUB=%d %.1f Gweight/s  %.2f weight/clk/SM @1965  %s\n", name, UPL, SUB, weights / ms / 1e6,
         weights / (ms * 1e-3) / 148.0 / 1.965e9, cudaGetErrorString(e));
  cudaFree(R); cudaFree(out);
}

int main() {
  run<4, 0, 16>("base");
  run<4, 1, 16>("fh-shfl3");
  run<4, 2, 16>("fh-lds128");
  run<4, 3, 16>("fh-mix");
  run<4, 4, 16>("fh-lea");
  run<2, 0, 16>("base");
  run<2, 2, 16>("fh-lds128");
  run<2, 3, 16>("fh-mix");
  run<4, 2, 8>("fh-lds128");
  run<4, 3, 8>("fh-mix");
  return 0;
}
