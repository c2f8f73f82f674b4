// tools/micro/fhash2.cu -- round-2 ceiling of the decode inner loop (tuning aid, not product).
// The loop of k_gemv_fast (DESIGN.md 2.2 hash, bank-private cells, 16-row subtiles, transpose
// butterfly) with variants of the select + multiply and of where the row mixes come from:
//   MODE 0: product form of round 1 -- rho words, VIMNMX3 + SHF (rotr) + FFMA, R from a per-warp
//           shared table (LDS.128 per row) filled per subtile
//   MODE 1: bf16 "key|value" words (high half = rho16 key, low half = bf16 bits): VIMNMX3 picks
//           the word, FHFMA.BF16 (fma.rn.f32.bf16) multiplies its low half by bf16 x -- no SHF
//   MODE 2: as 1, R from the global position table (LDG.128, L1-resident) -- no table fill
//   MODE 3: as 2, row 2's address from IMAD instead of the LOP3 mask form
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fh2 tools/micro/fhash2.cu && ./fh2
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t lds(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ float fmab(uint32_t xh, uint32_t w, float c) {  // c + bf16(x) * bf16(low half of w)
  float d;
  asm("{.reg .b16 lo, hi, xl, xh2; mov.b32 {lo, hi}, %2; mov.b32 {xl, xh2}, %1;\n\t"
      "fma.rn.f32.bf16 %0, xl, lo, %3;}"
      : "=f"(d) : "r"(xh), "r"(w), "f"(c));
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

template <int UPL, int MODE, int SUB, int THREADS, int MAXREG>
__global__ void __launch_bounds__(THREADS, 1) __maxnreg__(MAXREG)
    kern(const uint4* __restrict__ Rg, float* out, int rows_per_warp, int N, int nrt) {
  extern __shared__ __align__(128) uint32_t sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int maxN = N + 1, maxMN = 3 * maxN;
  const int cells = UPL * 32 * maxMN;
  for (int i = threadIdx.x; i < cells; i += blockDim.x) sm[i] = (i * 2654435761u) & 0x7FFF7FFFu;
  uint4* rt = reinterpret_cast<uint4*>(sm + cells + 64) + warp * SUB;  // per-warp R table
  const uint32_t smb = (uint32_t)__cvta_generic_to_shared(sm);
  const uint32_t rtb = (uint32_t)__cvta_generic_to_shared(rt);
  __syncthreads();
  uint32_t fk[UPL][3], cb[UPL][3], B = smb + 4u * lane;
  float Nf[UPL], Nf128[UPL], nx[UPL];
  uint32_t xb[UPL];
  for (int v = 0; v < UPL; ++v) {
    const uint32_t K = 0x12345u * (v + 1) + lane * 77u;
    for (int i = 0; i < 3; ++i) {
      fk[v][i] = ((K * (2 * i + 7)) & 0x7FFFFFu) | 0x3F800000u;
      cb[v][i] = __float_as_uint((float)(33554432 - 4 * N + 4 * (v * maxMN + i * maxN)));
    }
    Nf[v] = (float)(4 * N);
    Nf128[v] = (float)(128 * N);
    if (MODE == 1 || MODE == 2)  // row 2: LOP3 mask form (addend = 2^23 + byte address of the slot row - 128 N)
      cb[v][2] = __float_as_uint((float)(8388608u + smb + 128u * (uint32_t)(v * maxMN + 2 * maxN) - 128u * N));
    if (MODE == 0) cb[v][2] = __float_as_uint((float)(8388608u + smb + 128u * (uint32_t)(v * maxMN + 2 * maxN) - 128u * N));
    nx[v] = -(1.0f + v * 0.25f);
    xb[v] = 0x3F80u + v;
  }
  const uint32_t l4 = lane * 4u;
  float tot = 0.f;
  const uint4* Rw = Rg + (blockIdx.x * 97 + warp * 31) % (nrt - 4096);  // rows_per_warp <= 4096
  for (int s = 0; s < rows_per_warp; s += SUB) {
    if (MODE == 0 || MODE == 1) {  // per-subtile table fill (fmix of the row's position, 3 rows)
      __syncwarp();
      if (lane < SUB) {
        uint32_t o = (uint32_t)(s + lane) ^ 0x9E3779B9u;
        o ^= o >> 16; o *= 0x85EBCA6Bu; o ^= o >> 13; o *= 0xC2B2AE35u; o ^= o >> 16;
        uint32_t o2 = o * 0x2545F491u, o3 = o * 0x9E3779B9u;
        rt[lane] = make_uint4(o & 0x7FFFFFu, o2 >> 9, o3 >> 9, 0);
      }
      __syncwarp();
    }
    float acc[SUB];
#pragma unroll
    for (int r = 0; r < SUB; ++r) {
      uint4 q;
      if (MODE == 0 || MODE == 1)
        asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(q.x), "=r"(q.y), "=r"(q.z), "=r"(q.w) : "r"(rtb + 16u * r));
      else
        q = __ldg(Rw + s + r);
      float a = 0.f;
#pragma unroll
      for (int v = 0; v < UPL; ++v) {
        const uint32_t q0 = __float_as_uint(__fmaf_rz(__uint_as_float(q.x ^ fk[v][0]), Nf[v], __uint_as_float(cb[v][0])));
        const uint32_t q1 = __float_as_uint(__fmaf_rz(__uint_as_float(q.y ^ fk[v][1]), Nf[v], __uint_as_float(cb[v][1])));
        uint32_t m2;
        if (MODE == 3) {
          const uint32_t q2 = __float_as_uint(__fmaf_rz(__uint_as_float(q.z ^ fk[v][2]), Nf[v], __uint_as_float(cb[v][2])));
          m2 = lds(q2 * 128u + B);
        } else {
          const uint32_t q2 = __float_as_uint(__fmaf_rz(__uint_as_float(q.z ^ fk[v][2]), Nf128[v], __uint_as_float(cb[v][2])));
          uint32_t a2;
          asm("lop3.b32 %0, %1, 0x7FFF80, %2, 0xEA;" : "=r"(a2) : "r"(q2), "r"(l4));
          m2 = lds(a2);
        }
        const uint32_t m0 = lds(q0 * 128u + B), m1 = lds(q1 * 128u + B);
        const uint32_t b = max(max(m0, m1), m2);
        if (MODE == 0) a = fmaf(nx[v], __uint_as_float(__funnelshift_r(b, b, 1)), a);
        else a = fmab(xb[v], b, a);
      }
      acc[r] = a;
    }
    tot += transpose_reduce<SUB>(acc, lane);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = tot;
}

template <int UPL, int MODE, int SUB, int THREADS, int MAXREG>
void run(const char* name, int N) {
  const size_t smem = (size_t)UPL * 32 * 3 * (N + 1) * 4 + 256 + 16 * (THREADS / 32) * SUB + 128;
  cudaFuncSetAttribute(kern<UPL, MODE, SUB, THREADS, MAXREG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int grid = 148;
  const int nrt = 8192;
  uint4* R;
  float* out;
  cudaMalloc(&R, nrt * 16);
  {
    uint4* h = new uint4[nrt];
    for (int i = 0; i < nrt; ++i) {
      uint32_t o = (uint32_t)i * 0x9E3779B9u;
      o ^= o >> 15;
      h[i] = make_uint4(o & 0x7FFFFFu, (o * 0x2545F491u) >> 9, (o * 0x85EBCA77u) >> 9, 0);
    }
    cudaMemcpy(R, h, nrt * 16, cudaMemcpyHostToDevice);
    delete[] h;
  }
  cudaMalloc(&out, (size_t)grid * THREADS * 4);
  const int rows = 16 * 64 * 512 / THREADS;
  kern<UPL, MODE, SUB, THREADS, MAXREG><<<grid, THREADS, smem>>>(R, out, rows, N, nrt);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int it = 0; it < 10; ++it) kern<UPL, MODE, SUB, THREADS, MAXREG><<<grid, THREADS, smem>>>(R, out, rows, N, nrt);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  cudaError_t e = cudaGetLastError();
  const double weights = 10.0 * grid * THREADS * (double)rows * UPL;
  printf("%-22s UPL=%d SUB=%2d thr=%d reg=%d N=%3d %7.1f Gweight/s  %.2f weight/clk/SM @1965  %s\n", name, UPL, SUB,
         THREADS, MAXREG, N, weights / ms / 1e6, weights / (ms * 1e-3) / 148.0 / 1.965e9, cudaGetErrorString(e));
  cudaFree(R);
  cudaFree(out);
}

int main() {
  for (int N : {85, 21}) {
    run<4, 0, 16, 512, 112>("r1-product", N);
    run<4, 1, 16, 512, 112>("bf16-fhfma", N);
    run<4, 2, 16, 512, 112>("bf16-fhfma-ldgR", N);
    run<4, 3, 16, 512, 112>("bf16-fhfma-ldgR-imad2", N);
    run<4, 1, 8, 512, 112>("bf16-fhfma", N);
    run<4, 2, 8, 512, 112>("bf16-fhfma-ldgR", N);
    run<4, 2, 4, 512, 112>("bf16-fhfma-ldgR", N);
    run<4, 2, 16, 640, 96>("bf16-fhfma-ldgR", N);
  }
  return 0;
}
