// gemm.cu -- the prefill computation stage on the 5th-generation tensor cores.
//
// PAPER.md:183-189 (§3.1): decompression -> computation -> release.  After usk_linear has
// rebuilt the output-row slice W' [N, K] (bf16, K contiguous) into an L2-resident workspace,
// this kernel computes Y[T, N] = X[T, K] . W'^T with tcgen05.mma (kind::f16, bf16 x bf16 ->
// fp32 accumulation in TMEM).  DESIGN.md §Prefill explains why the reconstruction is not fused
// into the B-tile producer (CUDA-core reconstruction would be 2-3x slower than the MMA at
// 128-256-token reuse).
//
// Structure: persistent, one CTA (256 threads) per SM walks 128 x 256 output tiles
// (tile = blockIdx.x + k * gridDim.x, m fastest within groups of 8 n-blocks for L2 reuse):
//   warp 0      TMA producer: A tile [128 x 64] + B tile [256 x 64] per stage, SWIZZLE_128B,
//               4-stage ring guarded by full/empty mbarriers, flowing across tiles;
//   warp 1      MMA issuer (one elected lane): 4 x tcgen05.mma (K = 16 each) per stage into one of
//               TWO TMEM accumulators (tile parity), tcgen05.commit -> empty[stage]; after a
//               tile's last stage, commit -> acc_full[parity];
//   warp 2      TMEM allocator (512 fp32 columns = 2 x the 128 x 256 accumulator);
//   warps 4..7  epilogue: wait acc_full[parity], tcgen05.ld 32x32b (warp w reads TMEM lanes
//               32*(w%4)..+31 = its 32 output rows), convert, store, then release the accumulator
//               (acc_empty[parity]) -- so the epilogue of tile i overlaps the MMAs of tile i+1.
//
// The default launch is the CTA-pair form of the same pipeline, k_gemm_tc2 (cta_group::2, 256 x 256
// tiles per cluster of two, 6 stages of 32 KB per CTA; see its comment).  USK_GEMM_1SM=1 selects
// the 1-CTA kernel above (A/B only).  Measured on one B200, Llama-3.2-1B block at T = 16384: 1.760
// vs 1.876 ms per block (tools/prefill_split.py); ncu on the gate GEMM: tensor pipe 84 % of active
// cycles, shared-memory pipe 77 %, SM clock 1.48 GHz under the power cap (profiles/r1_gemm2_ncu.txt).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "common.cuh"
#include "ptx.cuh"

namespace usk {
namespace {

constexpr int BM = 128, BN = 256, BK = 64;
constexpr int kGemmSegs = 8;
constexpr int kStages = 4;
constexpr int kGemmThreads = 256;
constexpr uint32_t kABytes = BM * BK * 2;  // 16 KB
constexpr uint32_t kBBytes = BN * BK * 2;  // 32 KB
constexpr uint32_t kStageBytes = kABytes + kBBytes;
constexpr uint32_t kTmemCols = 512;  // two 128 x 256 fp32 accumulators
constexpr size_t kGemmSmem = 1024 /*align slack*/ + kStages * kStageBytes + 256 /*barriers*/;

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

// tcgen05 shared-memory matrix descriptor: K-major, SWIZZLE_128B (8 rows x 128 B atoms,
// SBO = 1024 B between 8-row groups, LBO unused = 1), version 1 (sm100).
__device__ __forceinline__ uint64_t smem_desc_sw128(const void* p) {
  const uint32_t a = smem_u32(p);
  uint64_t d = 0;
  d |= (uint64_t)((a & 0x3FFFF) >> 4);        // start address [0,14)
  d |= (uint64_t)1 << 16;                      // LBO (ignored for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;            // SBO [32,46)
  d |= (uint64_t)1 << 46;                      // version = 1
  d |= (uint64_t)2 << 61;                      // SWIZZLE_128B
  return d;
}

// instruction descriptor, kind::f16: D = F32, A = B = BF16, both K-major, M = 128, N = 256
constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
                            ((uint32_t)(BM >> 4) << 24);

__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(kIdesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// two fp32 -> packed bf16 pair, round to nearest even (one F2FP; lo in the low half)
__device__ __forceinline__ uint32_t pack_bf16x2(uint32_t lo, uint32_t hi) {
  uint32_t d;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(__uint_as_float(hi)), "f"(__uint_as_float(lo)));
  return d;
}

__device__ __forceinline__ uint16_t f32_to_bf16_rne(float f) {
  const uint32_t b = __float_as_uint(f);
  if ((b & 0x7F800000u) == 0x7F800000u) return (uint16_t)((b >> 16) | ((b & 0xFFFFu) ? 0x40u : 0u));
  return (uint16_t)((b + 0x7FFFu + ((b >> 16) & 1u)) >> 16);
}

struct GemmArgs {
  int32_t y_bf16;
  int32_t group_n;  // n-blocks per raster group (host: as many as keep the group's B rows L2-resident)
  int64_t T, N, K;
  // output column segments (usk_linear_batch_tokens: the layers of one GEMM): columns
  // [seg_col[s], seg_col[s+1]) go to seg_y[s] with leading dimension seg_ld[s]; inner boundaries are
  // multiples of 32 (one epilogue chunk never straddles two outputs)
  int32_t nseg;
  int32_t pad;
  int64_t seg_col[kGemmSegs + 1];
  void* seg_y[kGemmSegs];
  int64_t seg_ld[kGemmSegs];
};

// the output of a 32-column chunk starting at col: destination element and valid columns
template <typename T>
__device__ __forceinline__ T* out_at(const GemmArgs& G, int64_t row, int64_t col, int& nvalid) {
  int s = 0;
  while (s + 1 < G.nseg && col >= G.seg_col[s + 1]) ++s;
  nvalid = (int)min((int64_t)32, G.seg_col[s + 1] - col);
  return reinterpret_cast<T*>(G.seg_y[s]) + row * G.seg_ld[s] + (col - G.seg_col[s]);
}

// tile index -> (m block, n block): groups of group_n n-blocks, n fastest inside a group, so the
// concurrent tiles share a few A (X) row blocks and the group's B (W') rows stay in L2 while the
// m blocks advance: X is read from HBM once per group (one group covers all of W' when W' fits)
__device__ __forceinline__ void tile_coords(int64_t t, int mblocks, int nblocks, int group_n, int& mb, int& nb) {
  const int64_t per_group = (int64_t)mblocks * group_n;
  const int g = (int)(t / per_group);
  const int64_t r = t - (int64_t)g * per_group;
  const int gw = min(group_n, nblocks - g * group_n);  // n-blocks in this group
  mb = (int)(r / gw);
  nb = g * group_n + (int)(r % gw);
}

__global__ void __launch_bounds__(kGemmThreads, 1)
    k_gemm_tc(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
              const __grid_constant__ GemmArgs G) {
  extern __shared__ uint8_t gsm_raw[];
  uint8_t* gsm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(gsm_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = gsm;                                   // kStages x 16 KB
  uint8_t* sB = gsm + kStages * kABytes;               // kStages x 32 KB
  uint64_t* full = reinterpret_cast<uint64_t*>(gsm + kStages * kStageBytes);
  uint64_t* empty = full + kStages;
  uint64_t* acc_full = empty + kStages;   // [2]
  uint64_t* acc_empty = acc_full + 2;     // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mblocks = (int)((G.T + BM - 1) / BM), nblocks = (int)((G.N + BN - 1) / BN);
  const int64_t tiles = (int64_t)mblocks * nblocks;
  const int nkb = (int)((G.K + BK - 1) / BK);

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 4);  // one arrival per epilogue warp
    }
    fence_mbar_init();
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapB)) : "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int64_t it = 0;  // global stage counter across tiles
      for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
        int mb, nb;
        tile_coords(t, mblocks, nblocks, G.group_n, mb, nb);
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = (int)(it % kStages);
          if (it >= kStages) mbar_wait(&empty[s], (uint32_t)((it / kStages) - 1) & 1u);
          mbar_arrive_expect_tx(&full[s], kStageBytes);
          tma_load_2d(sA + s * kABytes, &mapA, &full[s], kb * BK, mb * BM);
          tma_load_2d(sB + s * kBBytes, &mapB, &full[s], kb * BK, nb * BN);
        }
      }
    }
  } else if (warp == 1) {
    int64_t it = 0;
    int local = 0;
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x, ++local) {
      const int b = local & 1;
      if (local >= 2) mbar_wait(&acc_empty[b], (uint32_t)((local >> 1) - 1) & 1u);  // epilogue drained it
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t acc = tmem + (uint32_t)(b * BN);
      for (int kb = 0; kb < nkb; ++kb, ++it) {
        const int s = (int)(it % kStages);
        mbar_wait(&full[s], (uint32_t)(it / kStages) & 1u);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (lane == 0) {
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t da = smem_desc_sw128(sA + s * kABytes + k * 32);
            const uint64_t db = smem_desc_sw128(sB + s * kBBytes + k * 32);
            mma_bf16(acc, da, db, (kb | k) != 0);
          }
          mma_commit(&empty[s]);
          if (kb == nkb - 1) mma_commit(&acc_full[b]);
        }
        __syncwarp();
      }
    }
  } else if (warp >= 4) {
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    int local = 0;
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x, ++local) {
      const int b = local & 1;
      int mb, nb;
      tile_coords(t, mblocks, nblocks, G.group_n, mb, nb);
      mbar_wait(&acc_full[b], (uint32_t)(local >> 1) & 1u);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int64_t row = (int64_t)mb * BM + q * 32 + lane;
      const int64_t n0 = (int64_t)nb * BN;
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 32) {
        uint32_t r[32];
        tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(b * BN + c0), r);
        if (row >= G.T) continue;
        const int64_t col = n0 + c0;
        if (col >= G.N) continue;
        int nvalid;
        if (G.y_bf16) {
          uint16_t* dst = out_at<uint16_t>(G, row, col, nvalid);
          if (nvalid == 32 && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
#pragma unroll
            for (int v = 0; v < 4; ++v) {
              uint4 pk;
              pk.x = pack_bf16x2(r[8 * v + 0], r[8 * v + 1]);
              pk.y = pack_bf16x2(r[8 * v + 2], r[8 * v + 3]);
              pk.z = pack_bf16x2(r[8 * v + 4], r[8 * v + 5]);
              pk.w = pack_bf16x2(r[8 * v + 6], r[8 * v + 7]);
              reinterpret_cast<uint4*>(dst)[v] = pk;
            }
          } else {
            for (int v = 0; v < nvalid; ++v) dst[v] = f32_to_bf16_rne(__uint_as_float(r[v]));
          }
        } else {
          float* dst = out_at<float>(G, row, col, nvalid);
          if (nvalid == 32 && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
#pragma unroll
            for (int v = 0; v < 8; ++v)
              reinterpret_cast<uint4*>(dst)[v] = make_uint4(r[4 * v], r[4 * v + 1], r[4 * v + 2], r[4 * v + 3]);
          } else {
            for (int v = 0; v < nvalid; ++v) dst[v] = __uint_as_float(r[v]);
          }
        }
      }
      // all of this warp's TMEM reads of accumulator b are complete (tcgen05.wait::ld in tmem_ld32)
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[b]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 2) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols) : "memory");
  }
}

// ---------------------------------------------------------------------------------------------
// CTA-pair variant (cta_group::2): a cluster of two CTAs on one TPC computes a 256 x 256 tile with
// one tcgen05.mma (M = 256) issued by the leader CTA (rank 0).  CTA r stages A rows
// [256 m + 128 r, +128) and B rows [256 n + 128 r, +128) of each 64-wide K block (16 + 16 KB per
// stage), so each SM fills and the MMA reads half the B bytes of the 1-CTA kernel per flop: the
// 1-CTA 128 x 256 tile needs ~134 B/clk of shared-memory bandwidth per SM at the tensor peak (TMA
// writes + MMA operand reads), over the 128 B/clk an SM has; the pair needs ~90.
//   * full[s] lives in the leader: both CTAs' TMA loads (.cta_group::2) complete their bytes on it;
//     the leader posts the 64 KB expectation.
//   * the leader's commits are multicast to both CTAs: empty[s] (each CTA's producer reuses its own
//     half of stage s) and acc_full[b] (each CTA's epilogue drains its own TMEM: rows 128 r + lane).
//   * acc_empty[b] lives in the leader and counts the 8 epilogue warps of the pair.
constexpr int kStages2 = 6;
constexpr uint32_t kHalfBytes = 128 * BK * 2;        // 16 KB: one CTA's half of A or of B
constexpr uint32_t kStageBytes2 = 2 * kHalfBytes;     // per CTA
constexpr size_t kGemmSmem2 = 1024 + kStages2 * kStageBytes2 + 256;
// kind::f16, D = F32, A = B = BF16, K-major, M = 256 (pair), N = 256
constexpr uint32_t kIdesc2 = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(256 >> 3) << 17) |
                             ((uint32_t)(256 >> 4) << 24);

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of the same variable in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t map_rank(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, uint32_t leader_bar, int c0,
                                                 int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(leader_bar)
      : "memory");
}
__device__ __forceinline__ void mma_bf16_pair(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(kIdesc2), "r"(accumulate));
}
__device__ __forceinline__ void mma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}

__global__ void __launch_bounds__(kGemmThreads, 1)
    k_gemm_tc2(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
               const __grid_constant__ GemmArgs G) {
  extern __shared__ uint8_t gsm_raw[];
  uint8_t* gsm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(gsm_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = gsm;                                   // kStages2 x 16 KB
  uint8_t* sB = gsm + kStages2 * kHalfBytes;           // kStages2 x 16 KB
  uint64_t* full = reinterpret_cast<uint64_t*>(gsm + kStages2 * kStageBytes2);
  uint64_t* empty = full + kStages2;
  uint64_t* acc_full = empty + kStages2;  // [2]
  uint64_t* acc_empty = acc_full + 2;     // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const int mblocks = (int)((G.T + BM - 1) / BM), nblocks = (int)((G.N + BN - 1) / BN);
  const int mpairs = (mblocks + 1) / 2;
  const int64_t tiles = (int64_t)mpairs * nblocks;
  const int64_t pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  const int nkb = (int)((G.K + BK - 1) / BK);

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < kStages2; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 8);  // the 4 epilogue warps of each CTA of the pair
    }
    fence_mbar_init();
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapB)) : "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync_all();  // barriers of both CTAs initialised before any remote arrive / complete_tx
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  // programmatic dependent launch: the set-up above overlaps the previous kernel (the reconstruction
  // of W' into the workspace); X, W' and Y are touched only after it completed
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  if (warp == 0) {
    if (lane == 0) {
      int64_t it = 0;
      for (int64_t t = pair; t < tiles; t += npairs) {
        int mp, nb;
        tile_coords(t, mpairs, nblocks, G.group_n, mp, nb);
        const int arow = mp * 2 * BM + (int)rank * BM;
        const int brow = nb * BN + (int)rank * 128;
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = (int)(it % kStages2);
          if (it >= kStages2) mbar_wait(&empty[s], (uint32_t)((it / kStages2) - 1) & 1u);
          if (rank == 0) mbar_arrive_expect_tx(&full[s], 2 * kStageBytes2);
          const uint32_t lbar = map_rank(&full[s], 0);
          tma_load_2d_pair(sA + s * kHalfBytes, &mapA, lbar, kb * BK, arow);
          tma_load_2d_pair(sB + s * kHalfBytes, &mapB, lbar, kb * BK, brow);
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {
      int64_t it = 0;
      int local = 0;
      for (int64_t t = pair; t < tiles; t += npairs, ++local) {
        const int b = local & 1;
        if (local >= 2) mbar_wait(&acc_empty[b], (uint32_t)((local >> 1) - 1) & 1u);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t acc = tmem + (uint32_t)(b * BN);
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = (int)(it % kStages2);
          mbar_wait(&full[s], (uint32_t)(it / kStages2) & 1u);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          if (lane == 0) {
#pragma unroll
            for (int k = 0; k < BK / 16; ++k) {
              const uint64_t da = smem_desc_sw128(sA + s * kHalfBytes + k * 32);
              const uint64_t db = smem_desc_sw128(sB + s * kHalfBytes + k * 32);
              mma_bf16_pair(acc, da, db, (kb | k) != 0);
            }
            mma_commit_pair(&empty[s]);
            if (kb == nkb - 1) mma_commit_pair(&acc_full[b]);
          }
          __syncwarp();
        }
      }
    }
  } else if (warp >= 4) {
    const int q = warp & 3;
    const uint32_t leader_acc_empty[2] = {map_rank(&acc_empty[0], 0), map_rank(&acc_empty[1], 0)};
    int local = 0;
    for (int64_t t = pair; t < tiles; t += npairs, ++local) {
      const int b = local & 1;
      int mp, nb;
      tile_coords(t, mpairs, nblocks, G.group_n, mp, nb);
      mbar_wait(&acc_full[b], (uint32_t)(local >> 1) & 1u);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int64_t row = (int64_t)mp * 2 * BM + (int64_t)rank * BM + q * 32 + lane;
      const int64_t n0 = (int64_t)nb * BN;
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 32) {
        uint32_t r[32];
        tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(b * BN + c0), r);
        if (row >= G.T) continue;
        const int64_t col = n0 + c0;
        if (col >= G.N) continue;
        int nvalid;
        if (G.y_bf16) {
          uint16_t* dst = out_at<uint16_t>(G, row, col, nvalid);
          if (nvalid == 32 && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
#pragma unroll
            for (int v = 0; v < 4; ++v) {
              uint4 pk;
              pk.x = pack_bf16x2(r[8 * v + 0], r[8 * v + 1]);
              pk.y = pack_bf16x2(r[8 * v + 2], r[8 * v + 3]);
              pk.z = pack_bf16x2(r[8 * v + 4], r[8 * v + 5]);
              pk.w = pack_bf16x2(r[8 * v + 6], r[8 * v + 7]);
              reinterpret_cast<uint4*>(dst)[v] = pk;
            }
          } else {
            for (int v = 0; v < nvalid; ++v) dst[v] = f32_to_bf16_rne(__uint_as_float(r[v]));
          }
        } else {
          float* dst = out_at<float>(G, row, col, nvalid);
          if (nvalid == 32 && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
#pragma unroll
            for (int v = 0; v < 8; ++v)
              reinterpret_cast<uint4*>(dst)[v] = make_uint4(r[4 * v], r[4 * v + 1], r[4 * v + 2], r[4 * v + 3]);
          } else {
            for (int v = 0; v < nvalid; ++v) dst[v] = __uint_as_float(r[v]);
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive_remote(leader_acc_empty[b]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync_all();  // no remote arrive or MMA operand read targets a CTA that has exited
  if (warp == 2) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols) : "memory");
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

bool make_map(CUtensorMap* m, const void* base, int64_t rows, int64_t cols, int box_rows) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
  cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

usk_status launch_gemm_bf16(const void* X, const void* W, void* Y, int32_t y_dtype, int64_t T, int64_t n_out,
                            int64_t K, int64_t ldw, cudaStream_t st) {
  if (ldw != K) return fail(USK_EUNSUPPORTED, "tcgen05 path needs a dense W' (ldw == in_features)");
  const GemmOut out{Y, n_out, n_out};
  return launch_gemm_bf16_seg(X, W, &out, 1, y_dtype, T, K, st);
}

usk_status launch_gemm_bf16_seg(const void* X, const void* W, const GemmOut* outs, int nseg, int32_t y_dtype,
                                int64_t T, int64_t K, cudaStream_t st) {
  if ((K * 2) % 16 != 0)
    return fail(USK_EUNSUPPORTED, "tcgen05 path needs in_features % 8 == 0 (16-B TMA row pitch)");
  if (nseg < 1 || nseg > kGemmSegs) return fail(USK_EINVAL, "tcgen05 GEMM: 1..8 output segments");
  GemmArgs G{};
  G.y_bf16 = y_dtype == USK_BF16;
  G.T = T;
  G.K = K;
  G.nseg = nseg;
  int64_t n_out = 0;
  for (int s = 0; s < nseg; ++s) {
    if (s + 1 < nseg && outs[s].cols % 32 != 0)
      return fail(USK_EINVAL, "tcgen05 GEMM: inner output segments must have a multiple of 32 columns");
    G.seg_col[s] = n_out;
    G.seg_y[s] = outs[s].y;
    G.seg_ld[s] = outs[s].ld;
    n_out += outs[s].cols;
  }
  G.seg_col[nseg] = n_out;
  G.N = n_out;
  if ((reinterpret_cast<uintptr_t>(X) & 15) || (reinterpret_cast<uintptr_t>(W) & 15))
    return fail(USK_EINVAL, "tcgen05 path needs 16-B aligned operands");
  static const bool one_sm = [] {
    const char* e = std::getenv("USK_GEMM_1SM");
    return e && e[0] == '1';
  }();
  CUtensorMap ma, mb;
  if (!make_map(&ma, X, T, K, BM) || !make_map(&mb, W, n_out, K, one_sm ? BN : 128))
    return fail(USK_ECUDA, "cuTensorMapEncodeTiled failed");
  {
    // raster groups: the B rows of a group (group_n x 256 rows x K bf16) within ~48 MB of L2, so X is
    // read from HBM once per group (ncu, 1B gate [8192 x 2048], groups of 8: 300 MB DRAM reads for
    // 100 MB of operands -- X re-read per group as the 268 MB of Y stream through L2)
    static const int forced = [] { const char* e = std::getenv("USK_GEMM_GROUPN"); return e ? std::atoi(e) : 0; }();
    const int64_t nblocks = (n_out + BN - 1) / BN;
    const int64_t fit = std::max<int64_t>(8, (48ll << 20) / ((int64_t)BN * K * 2));
    G.group_n = forced > 0 ? forced : (int)std::min<int64_t>(nblocks, fit);
  }
  const int sms2 = device_sm_count();
  if (!one_sm) {
    USK_CUDA(ensure_smem((const void*)k_gemm_tc2, (int)kGemmSmem2));
    const int64_t mpairs = ((T + BM - 1) / BM + 1) / 2;
    const int64_t ptiles = mpairs * ((n_out + BN - 1) / BN);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(2 * std::min<int64_t>(ptiles, sms2 / 2)));
    cfg.blockDim = dim3(kGemmThreads);
    cfg.dynamicSmemBytes = kGemmSmem2;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    // PDL for the GEMM (its set-up under the reconstruction's tail) measured no gain on the config-4
    // pass (27.6 / 27.6 vs 27.4 / 27.1 ms, same box): opt-in only
    static const bool pdl = [] { const char* e = std::getenv("USK_GEMM_PDL"); return e && e[0] == '1'; }();
    cudaLaunchAttribute attr2[2] = {attr[0], {}};
    attr2[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr2[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr2;
    cfg.numAttrs = pdl ? 2 : 1;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, k_gemm_tc2, ma, mb, G);
    if (e != cudaSuccess) return fail(USK_ECUDA, cudaGetErrorString(e));
    USK_LAUNCHED("k_gemm_tc2");
    return USK_OK;
  }
  USK_CUDA(ensure_smem((const void*)k_gemm_tc, (int)kGemmSmem));
  const int sms = device_sm_count();
  const int64_t tiles = ((T + BM - 1) / BM) * ((n_out + BN - 1) / BN);
  k_gemm_tc<<<(unsigned)std::min<int64_t>(tiles, sms), kGemmThreads, kGemmSmem, st>>>(ma, mb, G);
  USK_LAUNCHED("k_gemm_tc");
  return USK_OK;
}

}  // namespace usk
