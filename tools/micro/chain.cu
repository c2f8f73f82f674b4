// tools/micro/chain.cu -- per-call synchronisation cost of the decode step's launch structure
// (tuning aid, not product).  64 dependent "calls" in one CUDA graph, each a split-K GEMV skeleton:
// a compute grid of one 512-thread CTA per SM (200 KB dynamic smem, like k_gemv_fast) that waits for
// its predecessor (griddepcontrol.wait), busy-works W ns, writes NPART partials per row; then the
// row sums.  Variants of how the sums are formed:
//   pair  : a second PDL-launched reduce kernel (round-1 product: k_gemv_fast + k_gemv_reduce)
//   none  : no reduction at all (lower bound of one launch per call)
//   last  : in-kernel -- every CTA bumps an arrival counter (release); the last one sums all rows
//   gbar  : in-kernel grid barrier (arrive + spin) then every CTA sums its slice of the rows
//   blk   : in-kernel, per row block: CTA c contributes partial slot c % 16 of row block c / 16 only;
//           the last of a block's contributors (acq_rel arrival counter) sums that block's rows
//   poll  : in-kernel, no atomics or fences: partials are stored as 8-byte {value, epoch} words
//           (single-copy atomic); CTA c writes slot c % 16 of row block c / 16, then sums 1/16 of
//           that block's rows after polling until all 16 slots carry this call's epoch
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o chain tools/micro/chain.cu && ./chain
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kRows = 4096, kPart = 16, kCalls = 64;

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

struct Args {
  const float* x;  // read after the wait (the dependency)
  float* part;     // [kRows][kPart]
  float* y;        // [kRows]
  unsigned* ctr;   // arrival counter of this call (zeroed by the graph's first node)
  int work_ns;
  int mode;
  const unsigned* rep;  // graph replay counter (epoch base)
  unsigned long long* ts;  // [148][4] globaltimer stamps of this call: start, work done, arrived, exit
  int fence;               // blk: 0 atom.acq_rel, 1 threadfence + relaxed atomicAdd, 2 no fence (timing only)
};

__global__ void __launch_bounds__(512, 1) kc(const __grid_constant__ Args A) {
  extern __shared__ uint32_t sm[];
  if (threadIdx.x == 0) sm[0] = 0;
  pdl_wait();
  pdl_trigger();
  const float xv = A.x[threadIdx.x & 255];
  const unsigned long long t0 = gt();
  if (threadIdx.x == 0) A.ts[blockIdx.x * 4 + 0] = t0;
  while (gt() - t0 < (unsigned long long)A.work_ns) {
  }
  // this CTA's partials: rows r with r % gridDim == blockIdx, all kPart slots (stand-in for chunk partials)
  if (A.mode != 4 && A.mode != 5)
    for (int e = blockIdx.x * 512 + threadIdx.x; e < kRows * kPart; e += gridDim.x * 512) A.part[e] = xv + e;
  if (A.mode == 2) {  // last CTA sums every row
    __shared__ unsigned last;
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned prev;
      asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], 1;" : "=r"(prev) : "l"(A.ctr) : "memory");
      last = (prev == gridDim.x - 1);
    }
    __syncthreads();
    if (last) {
      for (int r = threadIdx.x; r < kRows; r += 512) {
        float s = 0.f;
        for (int p = 0; p < kPart; ++p) s += __ldcg(A.part + r * kPart + p);
        A.y[r] = s;
      }
      if (threadIdx.x == 0) *A.ctr = 0;
    }
  } else if (A.mode == 4) {
    const int nblk = (gridDim.x + kPart - 1) / kPart, blk = blockIdx.x / kPart;
    const int rpb = (kRows + nblk - 1) / nblk, r0 = blk * rpb, r1 = min(kRows, r0 + rpb);
    const int nc = min(kPart, (int)gridDim.x - blk * kPart);  // contributors of this block
    for (int r = r0 + threadIdx.x; r < r1; r += 512) A.part[r * kPart + blockIdx.x % kPart] = xv + r;
    __shared__ unsigned last;
    __syncthreads();
    if (threadIdx.x == 0) {
      A.ts[blockIdx.x * 4 + 1] = gt();
      unsigned prev;
      if (A.fence == 0) {
        asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], 1;" : "=r"(prev) : "l"(A.ctr + blk) : "memory");
      } else if (A.fence == 1) {
        __threadfence();
        prev = atomicAdd(A.ctr + blk, 1u);
        __threadfence();
      } else {
        prev = atomicAdd(A.ctr + blk, 1u);
      }
      last = (prev == (unsigned)nc - 1);
      if (last) A.ctr[blk] = 0;
      A.ts[blockIdx.x * 4 + 2] = gt();
    }
    __syncthreads();
    if (last) {
      for (int r = r0 + threadIdx.x; r < r1; r += 512) {
        const float4* p = reinterpret_cast<const float4*>(A.part + r * kPart);
        float4 q[kPart / 4];
#pragma unroll
        for (int k = 0; k < kPart / 4; ++k) q[k] = __ldcg(p + k);
        float s = 0.f;
#pragma unroll
        for (int k = 0; k < kPart / 4; ++k) s += q[k].x + q[k].y + q[k].z + q[k].w;
        A.y[r] = s;
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) A.ts[blockIdx.x * 4 + 3] = gt();
  } else if (A.mode == 5) {
    const unsigned ep = *A.rep + 1u;
    const int nblk = (gridDim.x + kPart - 1) / kPart, blk = blockIdx.x / kPart, slot = blockIdx.x % kPart;
    const int rpb = (kRows + nblk - 1) / nblk, r0 = blk * rpb, r1 = min(kRows, r0 + rpb);
    const int nc = min(kPart, (int)gridDim.x - blk * kPart);
    unsigned long long* P = reinterpret_cast<unsigned long long*>(A.part);  // [kRows][kPart] {value, epoch}
    for (int r = r0 + threadIdx.x; r < r1; r += 512) {
      const float v = xv + r;
      const unsigned long long w = ((unsigned long long)ep << 32) | __float_as_uint(v);
      asm volatile("st.relaxed.gpu.u64 [%0], %1;" ::"l"(P + r * kPart + slot), "l"(w) : "memory");
    }
    // reduce this CTA's share of the block's rows
    const int share = (r1 - r0 + nc - 1) / nc, q0 = r0 + slot * share, q1 = min(r1, q0 + share);
    for (int r = q0 + threadIdx.x; r < q1; r += 512) {
      float s = 0.f;
      for (int p = 0; p < nc; ++p) {
        unsigned long long w;
        do {
          asm volatile("ld.relaxed.gpu.u64 %0, [%1];" : "=l"(w) : "l"(P + r * kPart + p) : "memory");
        } while ((unsigned)(w >> 32) != ep);
        s += __uint_as_float((unsigned)w);
      }
      A.y[r] = s;
    }
  } else if (A.mode == 3) {  // grid barrier, then a row slice per CTA
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned prev, cur;
      asm volatile("atom.add.release.gpu.u32 %0, [%1], 1;" : "=r"(prev) : "l"(A.ctr) : "memory");
      do {
        asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(cur) : "l"(A.ctr) : "memory");
      } while (cur < gridDim.x);
    }
    __syncthreads();
    for (int r = blockIdx.x * 512 + threadIdx.x; r < kRows; r += gridDim.x * 512) {
      float s = 0.f;
      for (int p = 0; p < kPart; ++p) s += __ldcg(A.part + r * kPart + p);
      A.y[r] = s;
    }
  }
}

__global__ void __launch_bounds__(256) kr(const __grid_constant__ Args A) {
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.x * 256 + threadIdx.x;
  if (r < kRows) {
    float s = 0.f;
    for (int p = 0; p < kPart; ++p) s += __ldcg(A.part + r * kPart + p);
    A.y[r] = s;
  }
}

__global__ void kbump(unsigned* rep) { *rep += 1u; }

__global__ void kzero(unsigned* c, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) c[i] = 0;
}

void launch(void* k, dim3 g, dim3 b, size_t smem, cudaStream_t st, const Args& A) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = g;
  cfg.blockDim = b;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  void* args[] = {(void*)&A};
  cudaLaunchKernelExC(&cfg, k, args);
}

int main() {
  const size_t smem = 200 * 1024;
  cudaFuncSetAttribute(kc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  float *x, *part, *y;
  unsigned* ctr;
  cudaMalloc(&x, 1024 * 4);
  cudaMemset(x, 0, 1024 * 4);
  cudaMalloc(&part, (size_t)kCalls * kRows * kPart * 8);
  cudaMemset(part, 0, (size_t)kCalls * kRows * kPart * 8);
  unsigned* rep;
  cudaMalloc(&rep, 4);
  cudaMemset(rep, 0, 4);
  cudaMalloc(&y, (size_t)kCalls * kRows * 4);
  cudaMalloc(&ctr, kCalls * 64 * 4);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  const char* names[] = {"pair", "none", "last", "gbar", "blk", "poll", "blk-tf", "blk-nofence"};
  unsigned long long* ts;
  cudaMalloc(&ts, (size_t)kCalls * 148 * 4 * 8);
  for (int work : {0, 5000}) {
    for (int mode : {0, 1, 4, 6, 7}) {
      cudaGraph_t g;
      cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
      kzero<<<kCalls, 64, 0, st>>>(ctr, kCalls * 64);
      kbump<<<1, 1, 0, st>>>(rep);
      for (int c = 0; c < kCalls; ++c) {
        const int m = mode >= 6 ? 4 : mode;
        Args A{c ? y + (size_t)(c - 1) * kRows : x, part + (size_t)c * kRows * kPart * 2, y + (size_t)c * kRows, ctr + 64 * c,
               work, m, rep, ts + (size_t)c * 148 * 4, mode == 6 ? 1 : mode == 7 ? 2 : 0};
        launch((void*)kc, dim3(148), dim3(512), smem, st, A);
        if (mode == 0) launch((void*)kr, dim3(kRows / 256), dim3(256), 0, st, A);
      }
      cudaStreamEndCapture(st, &g);
      cudaGraphExec_t ge;
      if (cudaGraphInstantiate(&ge, g, 0) != cudaSuccess) {
        printf("instantiate failed\n");
        return 1;
      }
      for (int i = 0; i < 3; ++i) cudaGraphLaunch(ge, st);
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a, st);
      const int reps = 20;
      for (int i = 0; i < reps; ++i) cudaGraphLaunch(ge, st);
      cudaEventRecord(b, st);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("%-11s work=%5d ns: %.2f us per call (%s)\n", names[mode], work, ms * 1e3 / reps / kCalls,
             cudaGetErrorString(cudaGetLastError()));
      if (mode >= 4) {  // breakdown from the last replay's stamps (calls 1..63)
        static unsigned long long h[kCalls * 148 * 4];
        cudaMemcpy(h, ts, sizeof(h), cudaMemcpyDeviceToHost);
        double work_to_arr = 0, arr = 0, red = 0, gap = 0;
        int n = 0;
        for (int c = 1; c < kCalls; ++c) {
          unsigned long long s0 = ~0ull, wmax = 0, amax = 0, emax = 0, prev_e = 0;
          for (int b = 0; b < 148; ++b) {
            const unsigned long long* t = h + ((size_t)c * 148 + b) * 4;
            s0 = t[0] < s0 ? t[0] : s0;
            wmax = t[1] > wmax ? t[1] : wmax;
            amax = t[2] > amax ? t[2] : amax;
            emax = t[3] > emax ? t[3] : emax;
            const unsigned long long* tp = h + ((size_t)(c - 1) * 148 + b) * 4;
            prev_e = tp[3] > prev_e ? tp[3] : prev_e;
          }
          work_to_arr += 0; arr += (double)(amax - wmax); red += (double)(emax - amax); gap += (double)(s0 - prev_e); ++n;
        }
        printf("    breakdown (us): last work-done -> last arrival %.2f, -> last exit stamp %.2f, prev exit -> next start %.2f\n",
               arr / n / 1e3, red / n / 1e3, gap / n / 1e3);
      }
      cudaGraphExecDestroy(ge);
      cudaGraphDestroy(g);
    }
  }
  return 0;
}
