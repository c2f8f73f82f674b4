// micro_gather.cu -- ceiling of the sketch-query inner loop on this GPU (tuning aid, not product).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o micro_gather tools/micro_gather.cu && ./micro_gather
// Variants (all: 148*occ CTAs x 512 threads, UPL units per lane, 32-row subtiles, M = 3):
//   full   : LOP3 + 3 x (IMAD, IMAD.HI, LEA, LDS) + VIMNMX3 + SHF + FFMA per weight
//   hash   : same arithmetic, the "gather" replaced by the address itself (no LDS)
//   gather : LDS of precomputed-ish addresses (address = LEA of an IADD chain), no multiply
//   mul16  : 16-bit range reduction ((h*a_i) >> 16) * N >> 16 (IMAD instead of IMAD.HI)
//   mul16u : mul16 with one per-unit base and the row offset folded in (uniform row stride)
//   hiaddr : q = mulhi(h*a_i, N*128) + R_vi (uniform row base in the IMAD.HI addend), address =
//            (q & ~127) | lane*4 (one LOP3): same index as mulhi(h*a_i, N), LEA moved to the ALU
//   oraddr : power-of-two aligned (unit, row) regions: address = base_vi_lane | (idx << 7)
//            (SHF + LOP3 on the ALU pipe instead of an IMAD/LEA)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int UPL, int MODE>
__global__ void __launch_bounds__(512) kern(const uint32_t* __restrict__ Rg, float* out, int rows_per_warp, uint32_t a0,
                                            uint32_t a1, uint32_t a2, int N) {
  extern __shared__ uint32_t sm[];
  const int lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < UPL * 32 * 3 * N; i += blockDim.x) sm[i] = i * 2654435761u;
  __syncthreads();
  uint32_t K[UPL], rb[UPL][3];
  float nx[UPL];
  for (int v = 0; v < UPL; ++v) {
    K[v] = 0x12345u * (v + 1) + lane;
    for (int i = 0; i < 3; ++i)
      rb[v][i] = MODE == 6 ? (((uint32_t)(v * 3 + i) << 14) | (4u * lane)) : 4u * (uint32_t)(v * 32 * 3 * N + i * N * 32 + lane);
    nx[v] = 1.0f + v;
  }
  const char* base = reinterpret_cast<const char*>(sm);
  float tot = 0.f;
  for (int s = 0; s < rows_per_warp; s += 32) {
    const uint32_t Rl = Rg[(blockIdx.x * 512 + threadIdx.x + s) & 4095];
    float acc[32];
#pragma unroll
    for (int r = 0; r < 32; ++r) {
      const uint32_t Rv = __shfl_sync(0xffffffffu, Rl, r);
      float a = 0.f;
#pragma unroll
      for (int v = 0; v < UPL; ++v) {
        const uint32_t h = Rv ^ K[v];
        uint32_t m0, m1, m2;
        if (MODE == 0 || MODE == 1) {
          const uint32_t o0 = (__umulhi(h * a0, N) << 7) + rb[v][0];
          const uint32_t o1 = (__umulhi(h * a1, N) << 7) + rb[v][1];
          const uint32_t o2 = (__umulhi(h * a2, N) << 7) + rb[v][2];
          if (MODE == 0) {
            m0 = *reinterpret_cast<const uint32_t*>(base + o0);
            m1 = *reinterpret_cast<const uint32_t*>(base + o1);
            m2 = *reinterpret_cast<const uint32_t*>(base + o2);
          } else {
            m0 = o0; m1 = o1; m2 = o2;
          }
        } else if (MODE == 3) {
          const uint32_t o0 = ((((h * a0) >> 16) * N >> 16) << 7) + rb[v][0];
          const uint32_t o1 = ((((h * a1) >> 16) * N >> 16) << 7) + rb[v][1];
          const uint32_t o2 = ((((h * a2) >> 16) * N >> 16) << 7) + rb[v][2];
          m0 = *reinterpret_cast<const uint32_t*>(base + o0);
          m1 = *reinterpret_cast<const uint32_t*>(base + o1);
          m2 = *reinterpret_cast<const uint32_t*>(base + o2);
        } else if (MODE == 4) {
          const uint32_t o0 = ((((h * a0) >> 16) * N >> 16) << 7) + rb[v][0];
          const uint32_t o1 = ((((h * a1) >> 16) * N >> 16) + N) << 7;
          const uint32_t o2 = ((((h * a2) >> 16) * N >> 16) + 2 * N) << 7;
          m0 = *reinterpret_cast<const uint32_t*>(base + o0);
          m1 = *reinterpret_cast<const uint32_t*>(base + o1 + rb[v][0]);
          m2 = *reinterpret_cast<const uint32_t*>(base + o2 + rb[v][0]);
        } else if (MODE == 6) {
          // regions of 16 KB: base(v, i) = (v * 3 + i) << 14, lane * 4 in the low bits
          const uint32_t i0 = __umulhi(h * a0, N), i1 = __umulhi(h * a1, N), i2 = __umulhi(h * a2, N);
          uint32_t s0, s1, s2;
          asm("shl.b32 %0, %1, 7;" : "=r"(s0) : "r"(i0));
          asm("shl.b32 %0, %1, 7;" : "=r"(s1) : "r"(i1));
          asm("shl.b32 %0, %1, 7;" : "=r"(s2) : "r"(i2));
          uint32_t o0, o1, o2;
          asm("or.b32 %0, %1, %2;" : "=r"(o0) : "r"(s0), "r"(rb[v][0]));
          asm("or.b32 %0, %1, %2;" : "=r"(o1) : "r"(s1), "r"(rb[v][1]));
          asm("or.b32 %0, %1, %2;" : "=r"(o2) : "r"(s2), "r"(rb[v][2]));
          m0 = *reinterpret_cast<const uint32_t*>(base + o0);
          m1 = *reinterpret_cast<const uint32_t*>(base + o1);
          m2 = *reinterpret_cast<const uint32_t*>(base + o2);
        } else if (MODE == 5) {
          const uint32_t N128 = (uint32_t)N << 7, l4 = lane * 4u;
          const uint32_t q0 = __umulhi(h * a0, N128) + (uint32_t)(v * 32 * 3 * N * 4);
          const uint32_t q1 = __umulhi(h * a1, N128) + (uint32_t)(v * 32 * 3 * N * 4 + N * 128);
          const uint32_t q2 = __umulhi(h * a2, N128) + (uint32_t)(v * 32 * 3 * N * 4 + 2 * N * 128);
          m0 = *reinterpret_cast<const uint32_t*>(base + ((q0 & ~127u) | l4));
          m1 = *reinterpret_cast<const uint32_t*>(base + ((q1 & ~127u) | l4));
          m2 = *reinterpret_cast<const uint32_t*>(base + ((q2 & ~127u) | l4));
        } else {
          const uint32_t o = ((h & 63u) << 7);
          m0 = *reinterpret_cast<const uint32_t*>(base + o + rb[v][0]);
          m1 = *reinterpret_cast<const uint32_t*>(base + o + rb[v][1]);
          m2 = *reinterpret_cast<const uint32_t*>(base + o + rb[v][2]);
        }
        const uint32_t b = max(max(m0, m1), m2);
        a = fmaf(nx[v], __uint_as_float(__funnelshift_r(b, b, 1)), a);
      }
      acc[r] = a;
    }
#pragma unroll
    for (int r = 0; r < 32; ++r) tot += acc[r];
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = tot;
}

template <int UPL, int MODE>
void run(const char* name, int occ_target) {
  const int N = 85;
  const size_t smem = MODE == 6 ? (size_t)UPL * 3 * 16384 : (size_t)UPL * 32 * 3 * N * 4;
  cudaFuncSetAttribute(kern<UPL, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern<UPL, MODE>, 512, smem);
  int grid = 148 * (occ < occ_target ? occ : occ_target);
  uint32_t* R;
  float* out;
  cudaMalloc(&R, 4096 * 4);
  cudaMemset(R, 7, 4096 * 4);
  cudaMalloc(&out, (size_t)grid * 512 * 4);
  const int rows = 32 * 64;  // per warp
  kern<UPL, MODE><<<grid, 512, smem>>>(R, out, rows, 0x9E3779B1u, 0x85EBCA77u, 0xC2B2AE3Du, N);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int it = 0; it < 5; ++it)
    kern<UPL, MODE><<<grid, 512, smem>>>(R, out, rows, 0x9E3779B1u, 0x85EBCA77u, 0xC2B2AE3Du, N);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double weights = 5.0 * grid * 512.0 * rows * UPL;
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("%-8s UPL=%d occ=%d grid=%d  %.1f Gweight/s  %.2f weight/clk/SM (at %.0f MHz)\n", name, UPL, occ, grid,
         weights / ms / 1e6, weights / (ms * 1e-3) / 148.0 / (clk * 1e3), clk / 1e3);
  cudaFree(R);
  cudaFree(out);
}

int main() {
  run<4, 6>("oraddr", 4);
  run<2, 6>("oraddr", 4);
  run<4, 3>("mul16", 4);
  run<4, 0>("full", 4);
  run<4, 1>("hash", 4);
  run<4, 2>("gather", 4);
  run<2, 0>("full", 4);
  run<2, 1>("hash", 4);
  run<2, 2>("gather", 4);
  run<1, 0>("full", 4);
  run<4, 0>("full", 1);
  return 0;
}
