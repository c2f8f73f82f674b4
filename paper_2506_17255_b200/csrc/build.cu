// build.cu -- K2: the sketch build ("AbsMin Scatter").
//
// Definition (Eq. 3-4; ledger L2/L4): cell S[u, i, c] holds the weight of
// minimum |.| among those whose hash in row i is c (ties -> the non-negative one), +Inf if none.
// On 32-bit keys kappa = rotl(bits_hi, 1) = (mag << 1) | sign this is a plain integer min, so
// atomicMin gives the same bytes for every interleaving.
//
// Fast path (ROW granularity, one input dimension per unit -- DESIGN.md L6):
//   * one CTA per tile of TJ = 32*UPL consecutive units (input dims) of a layer, all outputs
//     (no cross-CTA merge); a whole model is one launch so tiles balance across waves;
//   * warp 0 streams [32 rows x TJ] weight tiles into a 6-stage shared-memory ring with
//     cp.async.bulk + mbarrier (TMA bulk engine);
//   * 16 consumer warps (2 rows of each stage): lane L owns units UPL*L .. UPL*L+UPL-1; its
//     keys live in shared memory at word (v * 32 * maxMN + k * 32 + L), i.e. always in bank L,
//     so the M random bucket updates of a warp are bank-conflict free; each update is an
//     unconditional red.shared.min (see key_min).  Per weight row o the warp's lane i computes the
//     position mix R_i(o) and SHFL broadcasts it; the short-unit index and the
//     key's shared address come from one FFMA.RZ + one IMAD (short_fma_bits);
//   * the CTA then writes its units' cells (states, +Inf for empty) to the sketch.
// Generic path (LAYER granularity, dims_per_unit > 1, odd shapes, oversize units): keys are
// kept in place in the sketch buffer (32-bit atomicMin for fp32 cells, 16-bit CAS for bf16),
// then converted to states.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>
#include <type_traits>

#include <cub/device/device_radix_sort.cuh>

#include "common.cuh"
#include "ptx.cuh"

namespace usk {
namespace {

#ifndef USK_BUILD_ROWS
#define USK_BUILD_ROWS 64
#endif
constexpr int kRO = USK_BUILD_ROWS;  // weight rows per stage (each consumer warp takes kRO / 16 of them)
#ifndef USK_BUILD_CONSUMERS
#define USK_BUILD_CONSUMERS 16
#endif
constexpr int kConsumers = USK_BUILD_CONSUMERS;  // consumer warps (kRO / kConsumers rows of every stage each)
#ifndef USK_BUILD_ROWS_SMALL
#define USK_BUILD_ROWS_SMALL 256
#endif
// rows per stage by units per lane: 2- and 1-unit tiles (wide-key layers, e.g. Llama-3-8B gate/up) take
// 256 rows, spreading the per-row cost over as many weights (8B build 6.6 -> 5.0 ms at 128 rows,
// 4.85 at 256); 4-unit tiles keep 64 (0.66 vs 0.78 ms at 128 for the 1B model)
template <int UPL>
constexpr int ro_of() { return UPL <= 2 ? USK_BUILD_ROWS_SMALL : kRO; }
inline int ro_host(int upl) { return upl <= 2 ? USK_BUILD_ROWS_SMALL : kRO; }
static_assert(kRO % kConsumers == 0 && USK_BUILD_ROWS_SMALL % kConsumers == 0,
              "rows per stage must divide over the consumer warps");
constexpr int kBuildThreads = 32 * (kConsumers + 1);
// layers per launch.  Launches group layers of similar key size (tasks are sorted by out): one grid
// of all 112 Llama-3.2-1B layers sizes every CTA's keys for gate/up and measured 0.89 vs 0.80 ms
constexpr int kMaxTasks = 48;
constexpr size_t kSmemLimit = 227 * 1024;

struct alignas(64) BuildTask {
  CUtensorMap map;     // W as a 2-D tensor [out rows, in cols], box = 32 rows x TJ units (TMA tiles)
  const void* W;
  int64_t out, in;
  int64_t unit_base;   // global unit id of the layer's first unit
  int32_t tile_begin;  // first CTA of this task
  int32_t pad;
  int64_t qchunk0;     // query layout: global index of the layer's first chunk
  int32_t qcw;         //   and its chunk width (units)
  int32_t qtab;        //   table-driven layer (class order, ledger L34): chunk per key group from qg
};

struct BuildArgs {
  BuildTask task[kMaxTasks];
  int32_t n_tasks;
  int32_t M;
  int32_t maxMN;
  HashConsts hc;
  const int32_t* ncols;
  const uint8_t* nrows;  // M_u per unit (ledger L30: per-class rows; slot rows >= M_u are scratch)
  const int64_t* offsets;
  const uint32_t* ukeys;
  const uint4* R4;  // {R_0, R_1, R_2} mod 2^23 per output row (fast hash, M <= 3)
  void* sketch;
  int* err;
  uint32_t kap_max;  // largest accepted weight key: 0xFEFFFFFF (finite), 0xFF000000 (+Inf = excluded outlier)
  int32_t stages;    // ring depth: as many stages as the shared memory left beside the keys holds (<= kMaxStages)
  // query layout (usk.h USK_LAYOUT_QUERY): write the tile's cells as rho16 words of its key groups'
  // chunk slices instead of unit-major cells (bf16 plans)
  unsigned char* qsketch;
  const int64_t* qc_off;
  const int32_t* qc_N;
  const int32_t* qc_aux;  // [4][chunks]: first query position, units, rows, width
  const int32_t* qg;      // [2][groups]: query position, chunk
  int64_t n_chunks, n_groups;
};

static_assert(sizeof(BuildArgs) <= 32764, "BuildArgs must fit the 32 KB kernel-parameter limit");

constexpr int kMaxStages = 16;   // ring depth cap (the mbarrier header holds 2 x 16 barriers)
constexpr int kMinStages = 3;
constexpr int kBuildHdr = 256;   // full[16] + empty[16] mbarriers

template <typename E, int UPL>
constexpr int stage_bytes() { return ro_of<UPL>() * 16 + ro_of<UPL>() * 32 * UPL * (int)sizeof(E); }

// kappa-min update of one shared key: an unconditional red.shared.min (no return value).  A
// plain-load pre-check would skip most atomics, but ptxas turns the predicated atomic into a branch
// per gather (serialising the gathers); measured on B200 the unconditional form is ~10% faster
// for the full Llama-3.2-1B build.
__device__ __forceinline__ void key_min(uint32_t saddr, uint32_t kap) {
  asm volatile("red.shared.min.u32 [%0], %1;" ::"r"(saddr), "r"(kap) : "memory");
}

// GK (grouped keys, USK-XG with one N per key group, ledger L32): the UPL units of a lane lie in one
// key group, so they share the hash and N -- one shared address per (row o, sketch row i) serves all
// UPL units.  Keys then live at word (kidx * UPL + v) * 32 + lane (kidx = i * N + c): unit v is the
// immediate offset v * 128 from the row's address, which one FFMA.RZ at ulp UPL * 128 and one IMAD give
// (the packed-decode form, tests/test_oracle_hash.py::test_packed_float_form for ulp 512).
template <typename E, int UPL, int MT, int HASH, bool GK = false>
__global__ void __launch_bounds__(kBuildThreads) k_build_fast(const __grid_constant__ BuildArgs A) {
  constexpr int ES = sizeof(E);
  constexpr int TJ = 32 * UPL;
  constexpr int ROWB = TJ * ES;
  const int S = A.stages;  // ring depth (host: as many stages as fit beside the keys)
  constexpr int STAGEB = stage_bytes<E, UPL>();
  constexpr int MR = MT > 0 ? MT : 8;
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + kMaxStages;
  uint8_t* stages = smem + kBuildHdr;
  uint32_t* keys = reinterpret_cast<uint32_t*>(stages + S * STAGEB);
  if constexpr (GK) {  // the grouped address form needs a 512-B aligned key base (host adds the slack)
    const uint32_t a = smem_u32(keys);
    keys += ((512u - (a & 511u)) & 511u) / 4u;
  }
  const uint32_t smem_keys = smem_u32(keys);
  // key of tile-local unit ul, cell kidx (= i * N_u + c)
  auto key_at = [&](int ul, int kidx) -> uint32_t {
    return GK ? keys[(kidx * UPL + ul % UPL) * 32 + ul / UPL] : keys[(ul % UPL) * (32 * A.maxMN) + kidx * 32 + ul / UPL];
  };

  const int b = blockIdx.x;
  int ti = 0;
  while (ti + 1 < A.n_tasks && A.task[ti + 1].tile_begin <= b) ++ti;
  const BuildTask& T = A.task[ti];
  const int64_t j0 = (int64_t)(b - T.tile_begin) * TJ;
  const int nu = (int)min((int64_t)TJ, T.in - j0);
  const int M = MT > 0 ? MT : A.M;
  constexpr int RO = ro_of<UPL>();  // weight rows per stage
  const int64_t n_it = (T.out + RO - 1) / RO;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int stride_v = 32 * A.maxMN;  // words per unit slot

  {
    const int nwords = TJ * A.maxMN + 32;  // + one dummy word per lane (ragged tiles)
    uint4* k4 = reinterpret_cast<uint4*>(keys);
    for (int i = threadIdx.x; i < nwords / 4; i += blockDim.x) k4[i] = make_uint4(~0u, ~0u, ~0u, ~0u);
    for (int i = (nwords / 4) * 4 + threadIdx.x; i < nwords; i += blockDim.x) keys[i] = ~0u;
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumers);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == 0) {
    // ---------------- producer: bulk-copy weight row segments into the ring
    // one 2-D TMA tile per stage (32 rows x TJ units; rows past `out` and units past `in` are
    // zero-filled) plus one bulk copy of the rows' position mixes
    if (lane == 0) {
      for (int64_t it = 0; it < n_it; ++it) {
        const int s = (int)(it % S);
        if (it >= S) mbar_wait(&empty[s], (uint32_t)((it / S) - 1) & 1u);
        const int64_t o0 = it * RO;
        const int rows = (int)min((int64_t)RO, T.out - o0);
        uint8_t* st = stages + s * STAGEB;
        mbar_arrive_expect_tx(&full[s], (uint32_t)rows * 16u + (uint32_t)(RO * ROWB));
        bulk_g2s(st, A.R4 + o0, (uint32_t)rows * 16u, &full[s]);  // the rows' position mixes
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                smem_u32(st + RO * 16)),
            "l"(reinterpret_cast<uint64_t>(&T.map)), "r"((int)j0), "r"((int)o0), "r"(smem_u32(&full[s]))
            : "memory");
      }
    }
  } else {
    // ---------------- consumers: warp cw takes rows cw and cw + 16 of every stage
    const int cw = warp - 1;
    if constexpr (GK && MT > 0 && HASH == USK_HASH_X) {
      constexpr uint32_t SLB = 128u * UPL;  // bytes per kidx row of a lane's UPL unit slots
      const bool valid0 = UPL * lane < nu;
      const int64_t u0 = T.unit_base + j0 + (valid0 ? UPL * lane : 0);
      const uint32_t Kg = A.ukeys[u0];
      const uint32_t Ng = valid0 ? (uint32_t)A.ncols[u0] : 1u;
      uint32_t fk[MT], cb[MT];
#pragma unroll
      for (int i = 0; i < MT; ++i) {
        fk[i] = short_fkey(row_key(Kg, A.hc.kap[i]));
        // SLB * 2^23 + B_i - SLB * N: result of the FFMA at ulp SLB, B_i = key base + i * N * SLB
        cb[i] = __float_as_uint(__ull2float_rz((unsigned long long)SLB * 8388608ull + smem_keys +
                                               (unsigned long long)i * Ng * SLB - (unsigned long long)SLB * Ng));
      }
      const float NS = (float)(SLB * Ng);
      // bits * SLB keeps (biased exponent << 23) * SLB mod 2^32 (zero for SLB 512 / 256, 2^30 for 128)
      constexpr uint32_t EXP = 127u + 23u + (SLB == 512u ? 9u : SLB == 256u ? 8u : 7u);
      const uint32_t LB = 4u * (uint32_t)lane - (EXP << 23) * SLB;
      uint32_t kmax = 0;
      int s = 0;
      uint32_t ph = 0;
      for (int64_t it = 0; it < n_it; ++it) {
        mbar_wait(&full[s], ph);
        const uint8_t* st = stages + s * STAGEB;
        const int64_t o0 = it * RO;
        const int rows = (int)min((int64_t)RO, T.out - o0);
        constexpr int RR = RO / kConsumers;
        // every row's weights and position mixes are loaded before any update (the atomics' asm
        // "memory" clobbers would otherwise keep the next row's shared loads behind them); rows past
        // a partial last stage read the (zero-filled / stale) ring and are skipped at the update
        using WT = typename std::conditional<ES * UPL == 8, uint2,
                   typename std::conditional<ES * UPL == 16, uint4,
                   typename std::conditional<ES * UPL == 4, uint32_t, uint16_t>::type>::type>::type;
        WT wv[RR];
        uint4 R4v[RR];
#pragma unroll
        for (int rr = 0; rr < RR; ++rr) {
          const int r = cw + rr * kConsumers;
          wv[rr] = reinterpret_cast<const WT*>(st + RO * 16 + r * ROWB)[lane];
          R4v[rr] = reinterpret_cast<const uint4*>(st)[r];  // broadcast shared load
        }
#pragma unroll
        for (int rr = 0; rr < RR; ++rr) {
          const int r = cw + rr * kConsumers;
          if (r >= rows) break;
          uint32_t kap[UPL];
          if constexpr (ES == 2 && UPL == 4) {
            kap[0] = rotl1(wv[rr].x << 16);
            kap[1 % UPL] = rotl1(wv[rr].x & 0xFFFF0000u);
            kap[2 % UPL] = rotl1(wv[rr].y << 16);
            kap[3 % UPL] = rotl1(wv[rr].y & 0xFFFF0000u);
          } else if constexpr (ES == 2 && UPL == 2) {
            kap[0] = rotl1((uint32_t)wv[rr] << 16);
            kap[1 % UPL] = rotl1((uint32_t)wv[rr] & 0xFFFF0000u);
          } else if constexpr (ES == 2) {
            kap[0] = rotl1((uint32_t)wv[rr] << 16);
          } else if constexpr (UPL == 4) {
            kap[0] = rotl1(wv[rr].x);
            kap[1 % UPL] = rotl1(wv[rr].y);
            kap[2 % UPL] = rotl1(wv[rr].z);
            kap[3 % UPL] = rotl1(wv[rr].w);
          } else if constexpr (UPL == 2) {
            kap[0] = rotl1(wv[rr].x);
            kap[1 % UPL] = rotl1(wv[rr].y);
          } else {
            kap[0] = rotl1((uint32_t)wv[rr]);
          }
#pragma unroll
          for (int v = 0; v < UPL; ++v) kmax = max(kmax, kap[v]);
          const uint32_t R23[3] = {R4v[rr].x, R4v[rr].y, R4v[rr].z};
#pragma unroll
          for (int i = 0; i < MT; ++i) {
            const uint32_t a =
                __float_as_uint(__fmaf_rz(__uint_as_float(R23[i] ^ fk[i]), NS, __uint_as_float(cb[i]))) * SLB + LB;
#pragma unroll
            for (int v = 0; v < UPL; ++v) key_min(a + 128u * v, kap[v]);  // missing units: scratch slots
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        if (++s == S) {
          s = 0;
          ph ^= 1u;
        }
      }
      if (kmax > A.kap_max) atomicOr(A.err, 1);  // NaN / Inf weight (USK_ENONFINITE)
    } else {
    constexpr bool FAST = MT > 0 && HASH == USK_HASH_X;  // short-unit FFMA.RZ form
    constexpr int KR = FAST ? MT : 1;
    uint32_t K[UPL], N[UPL];
    uint32_t rb[UPL][FAST ? 1 : MR];  // generic: byte offsets of (unit v, sketch row i) for this lane
    uint32_t fk[UPL][KR], cb[UPL][KR];  // fast: FFMA key and addend of (unit v, sketch row i)
    float Nf[UPL];
    const uint32_t kbase = smem_keys + 4u * (uint32_t)lane;  // (0x4C000000 << 7) wraps to 0
#pragma unroll
    for (int v = 0; v < UPL; ++v) {
      const int ul = UPL * lane + v;
      const bool valid = ul < nu;
      const int64_t u = T.unit_base + j0 + (valid ? ul : 0);
      K[v] = A.ukeys[u];
      // a missing unit of a ragged tile updates a private dummy word (never written back) with a
      // zero candidate, so the loop below needs no branch
      N[v] = valid ? (uint32_t)A.ncols[u] : 1u;
      Nf[v] = (float)(4u * N[v]);
      if constexpr (FAST) {
#pragma unroll
        for (int i = 0; i < MT; ++i) {
          fk[v][i] = short_fkey(row_key(K[v], A.hc.kap[i]));
          cb[v][i] = short_cbits(N[v], valid ? (uint32_t)(v * A.maxMN + i * (int)N[v]) : (uint32_t)(UPL * A.maxMN));
        }
      } else {
#pragma unroll
        for (int i = 0; i < MR; ++i)
          rb[v][i] = valid ? 4u * (uint32_t)(v * stride_v + i * (int)N[v] * 32 + lane)
                           : 4u * (uint32_t)(TJ * A.maxMN + lane);
      }
    }
    uint32_t kmax = 0;
    int s = 0;
    uint32_t ph = 0;
    for (int64_t it = 0; it < n_it; ++it) {
      mbar_wait(&full[s], ph);
      const uint8_t* st = stages + s * STAGEB;
      const int64_t o0 = it * RO;
      const int rows = (int)min((int64_t)RO, T.out - o0);
      constexpr int RR = RO / kConsumers;
      if (FAST && ES == 2 && UPL == 4 && rows == RO) {
        // a full stage: every row's weights and position mixes are loaded before any update, so the
        // shared-load latency of a row overlaps the previous rows' hashing and atomics
        uint2 w2[RR];
        uint4 R4v[RR];
#pragma unroll
        for (int rr = 0; rr < RR; ++rr) {
          const int r = cw + rr * kConsumers;
          w2[rr] = reinterpret_cast<const uint2*>(st + RO * 16 + r * ROWB)[lane];
          R4v[rr] = reinterpret_cast<const uint4*>(st)[r];  // broadcast
        }
#pragma unroll
        for (int rr = 0; rr < RR; ++rr) {
          const uint32_t bts[4] = {w2[rr].x << 16, w2[rr].x & 0xFFFF0000u, w2[rr].y << 16, w2[rr].y & 0xFFFF0000u};
          const uint32_t R23[3] = {R4v[rr].x, R4v[rr].y, R4v[rr].z};
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            const uint32_t kap = rotl1(bts[v]);
            kmax = max(kmax, kap);
#pragma unroll
            for (int i = 0; i < (MT > 0 ? MT : 1); ++i)
              key_min(short_fma_bits(R23[i], fk[v % UPL][i % KR], Nf[v % UPL], cb[v % UPL][i % KR]) * 128u + kbase, kap);
          }
        }
      } else {
#pragma unroll
        for (int rr = 0; rr < RO / kConsumers; ++rr) {
          const int r = cw + rr * kConsumers;
          if (r >= rows) break;
          const uint32_t o = (uint32_t)(o0 + r);
          const uint8_t* row = st + RO * 16 + r * ROWB;
          uint32_t bits[UPL];
          if constexpr (ES == 2 && UPL == 4) {
            const uint2 v2 = reinterpret_cast<const uint2*>(row)[lane];
            bits[0] = v2.x << 16;
            bits[1 % UPL] = v2.x & 0xFFFF0000u;
            bits[2 % UPL] = v2.y << 16;
            bits[3 % UPL] = v2.y & 0xFFFF0000u;
          } else if constexpr (ES == 2 && UPL == 2) {
            const uint32_t v2 = reinterpret_cast<const uint32_t*>(row)[lane];
            bits[0] = v2 << 16;
            bits[1 % UPL] = v2 & 0xFFFF0000u;
          } else if constexpr (ES == 2) {
            bits[0] = (uint32_t)reinterpret_cast<const uint16_t*>(row)[lane] << 16;
          } else if constexpr (UPL == 4) {
            const uint4 v4 = reinterpret_cast<const uint4*>(row)[lane];
            bits[0] = v4.x;
            bits[1 % UPL] = v4.y;
            bits[2 % UPL] = v4.z;
            bits[3 % UPL] = v4.w;
          } else if constexpr (UPL == 2) {
            const uint2 v2 = reinterpret_cast<const uint2*>(row)[lane];
            bits[0] = v2.x;
            bits[1 % UPL] = v2.y;
          } else {
            bits[0] = reinterpret_cast<const uint32_t*>(row)[lane];
          }
          if constexpr (FAST) {
            const uint4 R4 = reinterpret_cast<const uint4*>(st)[r];  // broadcast shared load
            const uint32_t R23[3] = {R4.x, R4.y, R4.z};
  #pragma unroll
            for (int v = 0; v < UPL; ++v) {
              const uint32_t kap = rotl1(bits[v]);  // missing units: zero-filled by the tensor copy
              kmax = max(kmax, kap);
  #pragma unroll
              for (int i = 0; i < MT; ++i) key_min(short_fma_bits(R23[i], fk[v][i], Nf[v], cb[v][i]) * 128u + kbase, kap);
            }
          } else {
  #pragma unroll
            for (int v = 0; v < UPL; ++v) {
              const uint32_t kap = rotl1(bits[v]);  // missing units: zero-filled by the tensor copy
              kmax = max(kmax, kap);
  #pragma unroll
              for (int i = 0; i < MR; ++i) {
                if (MT == 0 && i >= M) break;
                uint32_t idx;
                if constexpr (HASH == USK_HASH_X) idx = hash_index_x(A.hc, o, K[v], i, N[v]);
                else idx = o % N[v];
                key_min(smem_keys + rb[v][i] + (idx << 7), kap);
              }
            }
          }
        }
        }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if (++s == S) {
        s = 0;
        ph ^= 1u;
      }
    }
    if (kmax > A.kap_max) atomicOr(A.err, 1);  // NaN / Inf weight (USK_ENONFINITE)
    }
  }
  __syncthreads();

  if (ES == 2 && A.qsketch) {
    // ---------------- query layout: word (i, k, g) of the chunk = the 8 rho16 keys of key group g's
    // cell (i, k) (usk.h).  The tile holds groups [g_lo, g_lo + TJ / 8) of chunk j0 / 256; the layer's
    // last tile also writes the chunk's missing groups (zeros).  N_u and M_u of the tile's units are
    // staged in the idle ring first.
    int32_t* tN = reinterpret_cast<int32_t*>(stages);
    int32_t* tM = tN + TJ;
    for (int ul = threadIdx.x; ul < TJ; ul += blockDim.x) {
      const bool ok = ul < nu;
      tN[ul] = ok ? A.ncols[T.unit_base + j0 + ul] : 0;
      tM[ul] = ok ? (int)A.nrows[T.unit_base + j0 + ul] : 0;
    }
    __syncthreads();
    if (T.qtab) {
      // class-ordered layer (ledger L34): each key group of the tile goes to its own chunk / slot;
      // the group at a chunk's last query positions also writes the chunk's empty slots (zeros)
      const int ngt = (nu + kQGroup - 1) / kQGroup;
      for (int gg = 0; gg < ngt; ++gg) {
        const int64_t G = (T.unit_base + j0) / kQGroup + gg;
        const int qpos = A.qg[G];
        const int64_t a = A.qg[A.n_groups + G];
        const int q0 = A.qc_aux[a], na = A.qc_aux[A.n_chunks + a], Ma = A.qc_aux[2 * A.n_chunks + a];
        const int CWa = A.qc_aux[3 * A.n_chunks + a], maxN = A.qc_N[a];
        const int slot = (qpos - q0) / kQGroup, CWG = CWa / kQGroup;
        const bool lastg = qpos + kQGroup >= q0 + na;
        const int nz = lastg ? CWG - (slot + 1) : 0;  // empty slots after this group
        uint4* qo = reinterpret_cast<uint4*>(A.qsketch + A.qc_off[a]);
        const int64_t words = (int64_t)Ma * maxN;
        for (int64_t ik = threadIdx.x; ik < words * (1 + nz); ik += blockDim.x) {
          const int64_t sl = ik % words;
          const int extra = (int)(ik / words);  // 0: this group; 1..nz: the empty slots after it
          uint32_t w[4] = {0u, 0u, 0u, 0u};
          if (extra == 0) {
            const int i = (int)(sl / maxN), k = (int)(sl % maxN);
#pragma unroll
            for (int v8 = 0; v8 < kQGroup; ++v8) {
              const int ul = gg * kQGroup + v8;
              if (ul >= TJ) break;
              const int N = tN[ul];
              if (k < N && i < tM[ul]) {
                const uint32_t key = key_at(ul, i * N + k);
                const uint32_t b = (key == ~0u) ? 0x7F80u : (rotr1(key) >> 16);  // empty = +Inf
                w[v8 >> 1] |= ((((b << 1) | (b >> 15)) & 0xFFFFu) ^ 1u) << (16 * (v8 & 1));
              }
            }
          }
          qo[sl * CWG + slot + extra] = make_uint4(w[0], w[1], w[2], w[3]);
        }
      }
      return;
    }
    const int CWG = T.qcw / kQGroup;  // 16-B words (key groups) per slice of the chunk
    const int64_t chunk = j0 / T.qcw;
    const int g_lo = (int)((j0 % T.qcw) / kQGroup);
    const bool last = j0 + TJ >= T.in;
    const int g_hi = last ? CWG : g_lo + TJ / kQGroup;
    const int ng = g_hi - g_lo;
    const int maxN = A.qc_N[T.qchunk0 + chunk];
    uint4* qo = reinterpret_cast<uint4*>(A.qsketch + A.qc_off[T.qchunk0 + chunk]);
    const int64_t words = (int64_t)A.M * maxN * ng;
    for (int64_t e = threadIdx.x; e < words; e += blockDim.x) {
      const int gg = (int)(e % ng);
      const int64_t ik = e / ng;
      const int i = (int)(ik / maxN), k = (int)(ik % maxN);
      uint32_t w[4] = {0u, 0u, 0u, 0u};
#pragma unroll
      for (int v8 = 0; v8 < kQGroup; ++v8) {
        const int ul = gg * kQGroup + v8;
        if (ul >= TJ) break;
        const int N = tN[ul];
        if (k < N && i < tM[ul]) {
          const uint32_t key = key_at(ul, i * N + k);
          const uint32_t b = (key == ~0u) ? 0x7F80u : (rotr1(key) >> 16);  // empty = +Inf
          w[v8 >> 1] |= ((((b << 1) | (b >> 15)) & 0xFFFFu) ^ 1u) << (16 * (v8 & 1));
        }
      }
      qo[ik * CWG + g_lo + gg] = make_uint4(w[0], w[1], w[2], w[3]);
    }
    return;
  }
  // ---------------- write states.  The tile's units are consecutive in the sketch, so its cells are
  // ONE contiguous range [c0, c1).  Keys -> states into a staging copy of that range in the (now
  // idle) ring memory -- lane L reads its own units' keys (bank L, conflict-free) -- then one bulk
  // copy shared -> global for the 16-B aligned middle; the few cells of the unaligned head / tail go
  // out as plain stores.  (Per-lane stores straight from the keys would be 2-byte writes ~MN cells
  // apart: 32 sectors per warp store instruction.)
  E* out = reinterpret_cast<E*>(A.sketch);
  const int64_t c0 = A.offsets[T.unit_base + j0], c1 = A.offsets[T.unit_base + j0 + nu];
  const int64_t ncell = c1 - c0;
  const uint32_t lead = (uint32_t)((c0 * ES) & 15);  // staging byte offset = global byte address mod 16
  const bool staged = (size_t)ncell * ES + 16 <= (size_t)S * STAGEB;
  E* stg = reinterpret_cast<E*>(stages + lead);
#pragma unroll
  for (int v = 0; v < UPL; ++v) {
    const int ul = UPL * lane + v;
    if (ul >= nu) continue;
    const int64_t u = T.unit_base + j0 + ul;
    const int mn = (int)A.nrows[u] * A.ncols[u];  // the unit's own rows (<= M)
    const int64_t off = A.offsets[u];
    for (int k = warp; k < mn; k += kConsumers + 1) {
      const uint32_t key = key_at(ul, k);
      // empty = +Inf; Top-K builds (kap_max accepts the +Inf of excluded outliers):
      // a cell that only outliers (or nothing) map to holds +0 (DESIGN.md ledger L29)
      const uint32_t b32 = (A.kap_max >= 0xFF000000u && key >= 0xFF000000u) ? 0u
                           : (key == ~0u) ? 0x7F800000u : rotr1(key);
      const E cv = ES == 2 ? (E)(b32 >> 16) : (E)b32;
      if (staged) stg[off - c0 + k] = cv;
      else out[off + k] = cv;
    }
  }
  if (staged) {
    const int64_t g0 = c0 * ES, g1 = c1 * ES;              // tile byte range in the sketch
    const int64_t a0 = (g0 + 15) & ~int64_t(15), a1 = g1 & ~int64_t(15);
    fence_proxy_async_smem();                              // generic-proxy staging writes -> bulk copy
    __syncthreads();
    if (a1 > a0) {
      if (threadIdx.x == 0) {
        bulk_s2g(reinterpret_cast<uint8_t*>(A.sketch) + a0, stages + lead + (a0 - g0), (uint32_t)(a1 - a0));
        bulk_s2g_wait();                                   // complete before the CTA exits
      }
      for (int64_t c = c0 + threadIdx.x; c * ES < a0 && c < c1; c += blockDim.x) out[c] = stg[c - c0];
      for (int64_t c = a1 / ES + threadIdx.x; c < c1; c += blockDim.x) out[c] = stg[c - c0];
    } else {
      for (int64_t c = c0 + threadIdx.x; c < c1; c += blockDim.x) out[c] = stg[c - c0];
    }
  }
}

// ---------------------------------------------------------------- generic path
struct GenLayer {
  int64_t out, in, unit_base, cell_begin, n_cells;
  int32_t gran, g;
};

template <int ES>
__global__ void k_gen_init(void* sketch, int64_t c0, int64_t n) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (ES == 2) reinterpret_cast<uint16_t*>(sketch)[c0 + i] = 0xFFFF;
  else reinterpret_cast<uint32_t*>(sketch)[c0 + i] = 0xFFFFFFFFu;
}

__device__ __forceinline__ void cas_min16(uint16_t* cell, uint32_t key16) {
  uint32_t* word = reinterpret_cast<uint32_t*>(reinterpret_cast<uintptr_t>(cell) & ~uintptr_t(3));
  const int sh = (reinterpret_cast<uintptr_t>(cell) & 2) ? 16 : 0;
  uint32_t old = *reinterpret_cast<volatile uint32_t*>(word);
  for (;;) {
    const uint32_t cur = (old >> sh) & 0xFFFFu;
    if (key16 >= cur) return;
    const uint32_t nw = (old & ~(0xFFFFu << sh)) | (key16 << sh);
    const uint32_t prev = atomicCAS(word, old, nw);
    if (prev == old) return;
    old = prev;
  }
}

template <int ES, int HASH>
__global__ void k_gen_scatter(GenLayer G, const void* W, const uint8_t* nrows, HashConsts hc,
                              const int32_t* ncols, const int64_t* offsets, const uint32_t* ukeys,
                              void* sketch, int* err, uint32_t kap_max) {
  const int64_t n = G.out * G.in;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t o = e / G.in, j = e - o * G.in;
    int64_t t, p;
    unit_pos(G.gran, G.g, G.out, o, j, t, p);
    const int64_t u = G.unit_base + t;
    const uint32_t N = (uint32_t)ncols[u];
    const int64_t off = offsets[u];
    uint32_t bhi = (ES == 2) ? ((uint32_t)reinterpret_cast<const uint16_t*>(W)[e] << 16)
                             : reinterpret_cast<const uint32_t*>(W)[e];
    const uint32_t kap = rotl1(bhi);
    if (kap > kap_max) atomicOr(err, 1);
    const uint32_t Ku = ukeys[u];
    const int Mu = nrows[u];  // the unit's rows (ledger L30)
    for (int i = 0; i < Mu; ++i) {
      const uint32_t idx = (HASH == USK_HASH_X) ? hash_index_x(hc, (uint32_t)p, Ku, i, N) : (uint32_t)(p % N);
      const int64_t c = off + (int64_t)i * N + idx;
      if (ES == 2) {
        cas_min16(reinterpret_cast<uint16_t*>(sketch) + c, (kap >> 16) | (kap & 1u));  // kappa16 = (mag << 1) | s
      } else {
        uint32_t* cell = reinterpret_cast<uint32_t*>(sketch) + c;
        if (kap < *reinterpret_cast<volatile uint32_t*>(cell)) atomicMin(cell, kap);
      }
    }
  }
}

// keys -> states; empty = +Inf; zero_outlier_only (Top-K builds, DESIGN.md ledger
// L29): a cell whose min key is that of +Inf (only excluded outliers) or empty holds +0
template <int ES>
__global__ void k_gen_final(void* sketch, int64_t c0, int64_t n, int zero_outlier_only) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (ES == 2) {
    uint16_t* c = reinterpret_cast<uint16_t*>(sketch) + c0 + i;
    const uint32_t k = *c;
    *c = (zero_outlier_only && k >= 0xFF00u) ? (uint16_t)0
         : (k == 0xFFFFu) ? (uint16_t)0x7F80 : (uint16_t)((k >> 1) | ((k & 1u) << 15));
  } else {
    uint32_t* c = reinterpret_cast<uint32_t*>(sketch) + c0 + i;
    const uint32_t k = *c;
    *c = (zero_outlier_only && k >= 0xFF000000u) ? 0u : (k == 0xFFFFFFFFu) ? 0x7F800000u : ((k >> 1) | ((k & 1u) << 31));
  }
}

// ---------------------------------------------------------------- stacked state quantisation
// (scheme: SPEC.md quant module, DESIGN.md ledger L25)
template <int ES>
__global__ void k_fill_inf(void* raw, int64_t n) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (ES == 2) reinterpret_cast<uint16_t*>(raw)[i] = 0x7F80;  // empty = +Inf
  else reinterpret_cast<uint32_t*>(raw)[i] = 0x7F800000u;
}

// One warp per group of G cells (cell c = g*G + j, lane j mod 32): scale = fl32(absmax / qmax)
// over occupied (finite) cells, code = clamp(roundf(fl32(v / scale)), +-qmax) (round half away
// from zero), unoccupied cells and zero scales -> code 0.  Codes are stored packed: q = 8 one
// byte per cell, q = 4 two per byte with the even cell in the low nibble; scales as fp32.
template <int ES, int Q>
__global__ void k_quantize(const void* raw, int64_t g0, int64_t g1, int G, uint8_t* codes, float* scales) {
  const int64_t g = g0 + (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x & 31;
  if (g >= g1) return;  // uniform per warp
  const float qmax = Q == 4 ? 7.f : 127.f;
  auto value = [&](int64_t c) {
    return ES == 2 ? __uint_as_float((uint32_t)reinterpret_cast<const uint16_t*>(raw)[c] << 16)
                   : __uint_as_float(reinterpret_cast<const uint32_t*>(raw)[c]);
  };
  uint32_t amax = 0;  // bit pattern of max |v| (order-preserving for non-negative floats)
  for (int j = lane; j < G; j += 32) {
    const float v = value(g * G + j);
    if (isfinite(v)) amax = max(amax, __float_as_uint(fabsf(v)));
  }
  amax = __reduce_max_sync(0xffffffffu, amax);
  const float scale = __fdiv_rn(__uint_as_float(amax), qmax);
  if (lane == 0) scales[g] = scale;
  for (int j = lane; j < G; j += 32) {  // G % 32 == 0: every lane runs the same trip count
    const float v = value(g * G + j);
    int code = 0;
    if (isfinite(v) && scale > 0.f) code = (int)fminf(fmaxf(roundf(__fdiv_rn(v, scale)), -qmax), qmax);
    const int64_t c = g * G + j;
    if constexpr (Q == 8) {
      codes[c] = (uint8_t)(int8_t)code;
    } else {
      const int hi = __shfl_down_sync(0xffffffffu, code, 1);
      if ((lane & 1) == 0) codes[c >> 1] = (uint8_t)((code & 0xF) | ((hi & 0xF) << 4));
    }
  }
}

// ---------------------------------------------------------------- comparison variants
// (Appendix C.2; DESIGN.md ledger L27).  AbsMinMax keeps the max |.| per cell:
// keys rho = kappa ^ 1 = (mag << 1) | (1 - sign) (max rho = max |.|, ties -> non-negative), cells
// start at rho(+0) = 1.  bf16 cells hold the 16-bit rho16 = rotl16(bits, 1) ^ 1 (in-word CAS max).
__device__ __forceinline__ void cas_max16(uint16_t* cell, uint32_t key16) {
  uint32_t* word = reinterpret_cast<uint32_t*>(reinterpret_cast<uintptr_t>(cell) & ~uintptr_t(3));
  const int sh = (reinterpret_cast<uintptr_t>(cell) & 2) ? 16 : 0;
  uint32_t old = *reinterpret_cast<volatile uint32_t*>(word);
  for (;;) {
    const uint32_t cur = (old >> sh) & 0xFFFFu;
    if (key16 <= cur) return;
    const uint32_t nw = (old & ~(0xFFFFu << sh)) | (key16 << sh);
    const uint32_t prev = atomicCAS(word, old, nw);
    if (prev == old) return;
    old = prev;
  }
}

template <int ES>
__global__ void k_amx_init(void* sketch, int64_t c0, int64_t n) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (ES == 2) reinterpret_cast<uint16_t*>(sketch)[c0 + i] = 1;  // rho16(+0)
  else reinterpret_cast<uint32_t*>(sketch)[c0 + i] = 1u;         // rho(+0)
}

template <int ES, int HASH>
__global__ void k_amx_scatter(GenLayer G, const void* W, int32_t layer_M, HashConsts hc, const int32_t* ncols,
                              const int64_t* offsets, const uint32_t* ukeys, void* sketch, int* err) {
  const int64_t n = G.out * G.in;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t o = e / G.in, j = e - o * G.in;
    int64_t t, p;
    unit_pos(G.gran, G.g, G.out, o, j, t, p);
    const int64_t u = G.unit_base + t;
    const uint32_t N = (uint32_t)ncols[u];
    const int64_t off = offsets[u];
    const uint32_t bhi = (ES == 2) ? ((uint32_t)reinterpret_cast<const uint16_t*>(W)[e] << 16)
                                   : reinterpret_cast<const uint32_t*>(W)[e];
    const uint32_t kap = rotl1(bhi);
    if (kap >= 0xFF000000u) atomicOr(err, 1);
    const uint32_t rho = kap ^ 1u;
    const uint32_t Ku = ukeys[u];
    for (int i = 0; i < layer_M; ++i) {
      const uint32_t idx = (HASH == USK_HASH_X) ? hash_index_x(hc, (uint32_t)p, Ku, i, N) : (uint32_t)(p % N);
      const int64_t c = off + (int64_t)i * N + idx;
      if (ES == 2) {
        cas_max16(reinterpret_cast<uint16_t*>(sketch) + c, (rho >> 16) | (rho & 1u));
      } else {
        uint32_t* cell = reinterpret_cast<uint32_t*>(sketch) + c;
        if (rho > *reinterpret_cast<volatile uint32_t*>(cell)) atomicMax(cell, rho);
      }
    }
  }
}

template <int ES>
__global__ void k_amx_final(void* sketch, int64_t c0, int64_t n) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (ES == 2) {
    uint16_t* c = reinterpret_cast<uint16_t*>(sketch) + c0 + i;
    const uint32_t k = *c ^ 1u;  // kappa16 = (mag << 1) | sign
    *c = (uint16_t)((k >> 1) | ((k & 1u) << 15));
  } else {
    uint32_t* c = reinterpret_cast<uint32_t*>(sketch) + c0 + i;
    *c = rotr1(*c ^ 1u);
  }
}

// CountMin cells: fl32(fl64(S) * 2^-48) of the fixed-point sums, in the weight dtype (bf16: RNE)
template <int ES>
__global__ void k_cm_final(const unsigned long long* acc, int64_t n, void* sketch, int64_t c0) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float v = __double2float_rn(__ll2double_rn((long long)acc[i]) * (1.0 / 281474976710656.0));
  const uint32_t b = __float_as_uint(v);
  if (ES == 2) reinterpret_cast<uint16_t*>(sketch)[c0 + i] = (uint16_t)((b + 0x7FFFu + ((b >> 16) & 1u)) >> 16);
  else reinterpret_cast<uint32_t*>(sketch)[c0 + i] = b;
}

// ---------------------------------------------------------------- Top-K outliers
// (Appendix A; DESIGN.md ledger L29).  Selection key of weight e:
// (|w| bits << 32) | (2^32 - 1 - e): a descending sort ranks by |w|, ties -> smaller index.
__global__ void k_topk_keys(const void* W, int32_t es, int64_t n, unsigned long long* keys, int* err) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= n) return;
  uint32_t mag;
  if (es == 2) {
    const uint32_t b = reinterpret_cast<const uint16_t*>(W)[e];
    if ((b & 0x7F80u) == 0x7F80u) atomicOr(err, 1);
    mag = b & 0x7FFFu;
  } else {
    const uint32_t b = reinterpret_cast<const uint32_t*>(W)[e];
    if ((b & 0x7F800000u) == 0x7F800000u) atomicOr(err, 1);
    mag = b & 0x7FFFFFFFu;
  }
  keys[e] = ((unsigned long long)mag << 32) | (unsigned long long)(0xFFFFFFFFu - (uint32_t)e);
}

__global__ void k_topk_take(const unsigned long long* sorted, int64_t K, uint32_t* idx) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k < K) idx[k] = 0xFFFFFFFFu - (uint32_t)(sorted[k] & 0xFFFFFFFFull);
}

// side table (ascending flat indices, their states) + the outlier marked +Inf (= excluded) in
// the build copy of W
__global__ void k_topk_finish(const uint32_t* idx, int64_t K, const void* W, int32_t es, int32_t* tab_idx,
                              void* tab_vals, void* Wb) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= K) return;
  const uint32_t e = idx[k];
  tab_idx[k] = (int32_t)e;
  if (es == 2) {
    reinterpret_cast<uint16_t*>(tab_vals)[k] = reinterpret_cast<const uint16_t*>(W)[e];
    reinterpret_cast<uint16_t*>(Wb)[e] = 0x7F80;
  } else {
    reinterpret_cast<uint32_t*>(tab_vals)[k] = reinterpret_cast<const uint32_t*>(W)[e];
    reinterpret_cast<uint32_t*>(Wb)[e] = 0x7F800000u;
  }
}

// ---------------------------------------------------------------- host side
PFN_cuTensorMapEncodeTiled_v12000 encode_tiled() {
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

// W [rows, cols] row-major of es-byte elements; box = 32 rows x tj columns, no swizzle, zero fill.
// The encoding is a pure function of its arguments, so maps are cached by them (host, process-wide):
// repeated builds from the same weight buffers (a rebuild per training step, the bench's timed
// build) skip the ~1 us per layer host encode that otherwise delays the first launch.
bool make_w_map_uncached(CUtensorMap* m, const void* base, int64_t rows, int64_t cols, int es, int tj, int64_t ld);
bool make_w_map(CUtensorMap* m, const void* base, int64_t rows, int64_t cols, int es, int tj, int64_t ld = 0) {
  using Key = std::tuple<const void*, int64_t, int64_t, int, int, int64_t>;
  static std::mutex mu;
  static std::map<Key, CUtensorMap> cache;
  const Key key{base, rows, cols, es, tj, ld};
  {
    std::lock_guard<std::mutex> g(mu);
    auto it = cache.find(key);
    if (it != cache.end()) {
      *m = it->second;
      return true;
    }
  }
  if (!make_w_map_uncached(m, base, rows, cols, es, tj, ld)) return false;
  std::lock_guard<std::mutex> g(mu);
  if (cache.size() >= 4096) cache.clear();
  cache.emplace(key, *m);
  return true;
}

bool make_w_map_uncached(CUtensorMap* m, const void* base, int64_t rows, int64_t cols, int es, int tj, int64_t ld) {
  auto fn = encode_tiled();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld ? ld : cols) * es};
  cuuint32_t box[2] = {(cuuint32_t)tj, (cuuint32_t)ro_host(tj / 32)};
  cuuint32_t estr[2] = {1, 1};
  return fn(m, es == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base),
            dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int fast_upl(const usk_plan* pl, int32_t l, bool pitch_ok = false) {
  // units per lane for the fast kernels, 0 = not eligible: the largest UPL whose key array and
  // stage ring fit one CTA (one CTA per SM is enough: 17 warps, bulk-copy ring in flight).
  // pitch_ok: the caller pads the row pitch itself (row-sharded output-row builds)
  const LayerGeom& L = pl->layers[l];
  // output-row units (L31) build as input-dim units of W^T (the same sketch bytes, L31)
  const bool outrow = pl->gran == USK_GRAN_OUTROW;
  if ((pl->gran != USK_GRAN_ROW && !outrow) || pl->g != 1 || pl->variant != USK_ABSMAXMIN) return 0;
  const int es = pl->cell_bytes();
  if (!pitch_ok && ((outrow ? L.out : L.in) * es) % 16 != 0) return 0;
  const int64_t mn = (int64_t)pl->M * L.max_ncols;
  const int S = kMinStages;
  auto smem = [&](int upl) {
    const int64_t ro = ro_host(upl);
    return (int64_t)kBuildHdr + S * (ro * 16 + ro * 32 * upl * es) + 32LL * upl * mn * 4 + 128 + 512;
  };
  for (int upl : {4, 2, 1})
    if (smem(upl) <= (int64_t)kSmemLimit) return upl;
  return 0;
}

template <typename E, int UPL, int MT, int HASH, bool GK = false>
usk_status launch_fast_t(BuildArgs& A, int n_ctas, cudaStream_t st) {
  // ring depth: every stage the shared memory beside the keys holds (the bulk copies in flight per SM
  // must cover the HBM latency-bandwidth product: 3 stages of gate/up tiles are ~52 KB)
  const size_t keys = (size_t)32 * UPL * A.maxMN * 4 + 128 + (GK ? 512 : 0);
  static const int forced = [] { const char* e = std::getenv("USK_BUILD_STAGES"); return e ? std::atoi(e) : 0; }();
  int S = (int)std::min<size_t>(kMaxStages, (kSmemLimit - kBuildHdr - keys) / stage_bytes<E, UPL>());
  // grouped-key builds: 4 stages measured best (1B: 0.80 ms at 4, 0.81 at 3, 0.83 at 8, 0.84 at all
  // that fit) -- the consumers are latency-bound, a deeper ring only adds L2 pressure
  if (GK) S = std::min(S, 4);
  if (forced > 0) S = std::min(S, forced);
  if (S < kMinStages) return fail(USK_EINVAL, "usk_build: tile does not fit shared memory");
  A.stages = S;
  const size_t smem = kBuildHdr + (size_t)S * stage_bytes<E, UPL>() + keys;
  auto kern = k_build_fast<E, UPL, MT, HASH, GK>;
  USK_CUDA(ensure_smem((const void*)kern, 227 * 1024));  // one limit per (device, kernel): the opt-in maximum
  kern<<<n_ctas, kBuildThreads, smem, st>>>(A);
  USK_LAUNCHED("k_build_fast");
  return USK_OK;
}

template <typename E, int UPL>
usk_status launch_fast_m(BuildArgs& A, int n_ctas, int hash, cudaStream_t st, bool gk = false) {
  if (hash == USK_HASH_IDENTITY) return launch_fast_t<E, UPL, 0, USK_HASH_IDENTITY>(A, n_ctas, st);
  if (gk) {  // grouped keys (USK-XG, one N per key group)
    switch (A.M) {
      case 1: return launch_fast_t<E, UPL, 1, USK_HASH_X, true>(A, n_ctas, st);
      case 2: return launch_fast_t<E, UPL, 2, USK_HASH_X, true>(A, n_ctas, st);
      case 3: return launch_fast_t<E, UPL, 3, USK_HASH_X, true>(A, n_ctas, st);
      default: break;
    }
  }
  switch (A.M) {
    case 1: return launch_fast_t<E, UPL, 1, USK_HASH_X>(A, n_ctas, st);
    case 2: return launch_fast_t<E, UPL, 2, USK_HASH_X>(A, n_ctas, st);
    case 3: return launch_fast_t<E, UPL, 3, USK_HASH_X>(A, n_ctas, st);
    default: return launch_fast_t<E, UPL, 0, USK_HASH_X>(A, n_ctas, st);
  }
}

usk_status launch_fast(const usk_plan* pl, int upl, std::vector<std::pair<int32_t, const void*>>& group,
                       void* sketch, cudaStream_t st, uint32_t kap_max, void* qsketch = nullptr, bool gk = false) {
  // longest tasks first (largest out) so the big CTAs start in the first wave
  std::stable_sort(group.begin(), group.end(), [&](auto& a, auto& b) {
    return pl->layers[a.first].out > pl->layers[b.first].out;
  });
  for (size_t g0 = 0; g0 < group.size(); g0 += kMaxTasks) {
    BuildArgs A{};
    A.M = pl->M;
    A.hc = pl->hc;
    A.ncols = pl->d_ncols;
    A.nrows = pl->d_nrows;
    A.offsets = pl->d_offsets;
    A.ukeys = pl->d_keys;
    A.R4 = pl->d_R4;
    A.sketch = sketch;
    A.err = pl->d_err;
    A.kap_max = kap_max;
    A.qsketch = reinterpret_cast<unsigned char*>(qsketch);
    A.qc_off = pl->d_qc_off;
    A.qc_N = pl->d_qc_N;
    A.qc_aux = pl->d_qc_aux;
    A.qg = pl->d_qg;
    A.n_chunks = (int64_t)pl->h_qc_N.size();
    A.n_groups = (int64_t)pl->h_qperm.size();
    int tiles = 0, maxmn = 1;
    const int TJ = 32 * upl;
    for (size_t k = g0; k < std::min(group.size(), g0 + kMaxTasks); ++k) {
      const LayerGeom& L = pl->layers[group[k].first];
      BuildTask& t = A.task[A.n_tasks++];
      t.W = group[k].second;
      const bool outrow_t = pl->gran == USK_GRAN_OUTROW;
      if (!make_w_map(&t.map, t.W, outrow_t ? L.in : L.out, outrow_t ? L.out : L.in, pl->cell_bytes(), TJ))
        return fail(USK_ECUDA, "usk_build: cuTensorMapEncodeTiled failed");
      const bool outrow = pl->gran == USK_GRAN_OUTROW;  // W is W^T [in, out] here
      t.out = outrow ? L.in : L.out;
      t.in = outrow ? L.out : L.in;
      t.unit_base = L.unit_begin;
      t.qchunk0 = L.qchunk0;
      t.qcw = L.qcw;
      t.qtab = L.qperm;
      t.tile_begin = tiles;
      tiles += (int)((t.in + TJ - 1) / TJ);
      maxmn = std::max(maxmn, pl->M * L.max_ncols);
    }
    A.maxMN = maxmn;
    usk_status s;
    if (pl->dtype == USK_BF16)
      s = upl == 4   ? launch_fast_m<uint16_t, 4>(A, tiles, pl->hash, st, gk)
          : upl == 2 ? launch_fast_m<uint16_t, 2>(A, tiles, pl->hash, st, gk)
                     : launch_fast_m<uint16_t, 1>(A, tiles, pl->hash, st, gk);
    else
      s = upl == 4   ? launch_fast_m<uint32_t, 4>(A, tiles, pl->hash, st, gk)
          : upl == 2 ? launch_fast_m<uint32_t, 2>(A, tiles, pl->hash, st, gk)
                     : launch_fast_m<uint32_t, 1>(A, tiles, pl->hash, st, gk);
    if (s != USK_OK) return s;
  }
  return USK_OK;
}

// grouped-key build eligible: USK-XG keys and one N per key group in the layer (ledger L32), M <= 3
bool layer_gk_ok(const usk_plan* pl, int32_t l) {
  static const int off = [] { const char* e = std::getenv("USK_BUILD_GK"); return e ? std::atoi(e) == 0 : 0; }();
  if (off || pl->hash_api != USK_HASH_XG || pl->M > 3 || pl->gran != USK_GRAN_ROW) return false;
  return pl->layers[l].groups_one_n != 0;  // computed once with the plan
}

template <int ES>
usk_status launch_generic_t(const usk_plan* pl, int32_t l, const void* W, void* sketch, cudaStream_t st,
                            uint32_t kap_max = 0xFEFFFFFFu) {
  const LayerGeom& L = pl->layers[l];
  GenLayer G{L.out, L.in, L.unit_begin, L.cell_begin, L.n_cells, pl->gran, pl->g};
  const int T = 256;
  const unsigned cb = (unsigned)((std::max<int64_t>(L.n_cells, 1) + T - 1) / T);
  if (pl->variant == USK_COUNTMIN) {
    unsigned long long* acc = nullptr;
    USK_CUDA(cudaMallocAsync(&acc, (size_t)std::max<int64_t>(L.n_cells, 1) * 8, st));
    USK_CUDA(cudaMemsetAsync(acc, 0, (size_t)std::max<int64_t>(L.n_cells, 1) * 8, st));
    usk_status s = launch_fixed_accumulate(pl, l, W, pl->dtype, acc, pl->d_err, st);
    if (s == USK_OK && L.n_cells > 0) {
      k_cm_final<ES><<<cb, T, 0, st>>>(acc, L.n_cells, sketch, L.cell_begin);
      cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) s = cuda_fail(e, "k_cm_final");
      else count_launch();
    }
    cudaError_t e = cudaFreeAsync(acc, st);
    if (s == USK_OK && e != cudaSuccess) s = cuda_fail(e, "cudaFreeAsync");
    return s;
  }
  if (pl->variant == USK_ABSMINMAX) {
    k_amx_init<ES><<<cb, T, 0, st>>>(sketch, L.cell_begin, L.n_cells);
    USK_LAUNCHED("k_amx_init");
    const int64_t n = L.out * L.in;
    const unsigned blocks = (unsigned)std::min<int64_t>((n + T - 1) / T, 148 * 16);
    if (pl->hash == USK_HASH_X)
      k_amx_scatter<ES, USK_HASH_X><<<blocks, T, 0, st>>>(G, W, pl->M, pl->hc, pl->d_ncols, pl->d_offsets, pl->d_keys,
                                                          sketch, pl->d_err);
    else
      k_amx_scatter<ES, USK_HASH_IDENTITY><<<blocks, T, 0, st>>>(G, W, pl->M, pl->hc, pl->d_ncols, pl->d_offsets,
                                                                 pl->d_keys, sketch, pl->d_err);
    USK_LAUNCHED("k_amx_scatter");
    k_amx_final<ES><<<cb, T, 0, st>>>(sketch, L.cell_begin, L.n_cells);
    USK_LAUNCHED("k_amx_final");
    return USK_OK;
  }
  k_gen_init<ES><<<(unsigned)((L.n_cells + T - 1) / T), T, 0, st>>>(sketch, L.cell_begin, L.n_cells);
  USK_LAUNCHED("k_gen_init");
  const int64_t n = L.out * L.in;
  const unsigned blocks = (unsigned)std::min<int64_t>((n + T - 1) / T, 148 * 16);
  if (pl->hash == USK_HASH_X)
    k_gen_scatter<ES, USK_HASH_X><<<blocks, T, 0, st>>>(G, W, pl->d_nrows, pl->hc, pl->d_ncols, pl->d_offsets, pl->d_keys,
                                                        sketch, pl->d_err, kap_max);
  else
    k_gen_scatter<ES, USK_HASH_IDENTITY><<<blocks, T, 0, st>>>(G, W, pl->d_nrows, pl->hc, pl->d_ncols, pl->d_offsets,
                                                               pl->d_keys, sketch, pl->d_err, kap_max);
  USK_LAUNCHED("k_gen_scatter");
  k_gen_final<ES><<<(unsigned)((L.n_cells + T - 1) / T), T, 0, st>>>(sketch, L.cell_begin, L.n_cells,
                                                                     kap_max >= 0xFF000000u ? 1 : 0);
  USK_LAUNCHED("k_gen_final");
  return USK_OK;
}

}  // namespace

bool layer_fast_ok(const usk_plan* pl, int32_t l) { return fast_upl(pl, l) != 0; }

// W^T of a row-major [rows, cols] matrix of ES-byte elements (32 x 32 tiles through shared memory)
template <int ES>
__global__ void k_transpose(const void* src, void* dst, int64_t rows, int64_t cols, int64_t ld_dst) {
  using T = typename std::conditional<ES == 2, uint16_t, uint32_t>::type;
  __shared__ T tile[32][33];
  const int64_t c0 = (int64_t)blockIdx.x * 32, r0 = (int64_t)blockIdx.y * 32;
  const T* S = reinterpret_cast<const T*>(src);
  T* D = reinterpret_cast<T*>(dst);
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t r = r0 + i, c = c0 + threadIdx.x;
    if (r < rows && c < cols) tile[i][threadIdx.x] = S[r * cols + c];
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t c = c0 + i, r = r0 + threadIdx.x;
    if (r < rows && c < cols) D[c * ld_dst + r] = tile[threadIdx.x][i];
  }
}

static usk_status launch_build_raw(const usk_plan* pl, const void* const* weights, const int32_t* layer_ids,
                                   int32_t n, void* sketch, cudaStream_t st, uint32_t kap_max = 0xFEFFFFFFu) {
  std::vector<std::pair<int32_t, const void*>> grp[5];  // by units per lane (1, 2, 4)
  std::vector<std::pair<int32_t, const void*>> ggrp[5];  // grouped keys (USK-XG)
  std::vector<std::pair<int32_t, const void*>> tgrp[5];  // output-row units: built from W^T
  for (int32_t k = 0; k < n; ++k) {
    const int32_t l = layer_ids ? layer_ids[k] : k;
    const int upl = fast_upl(pl, l);
    if (upl) {
      (pl->gran == USK_GRAN_OUTROW ? tgrp : layer_gk_ok(pl, l) ? ggrp : grp)[upl].push_back({l, weights[k]});
    } else {
      usk_status s = pl->dtype == USK_BF16 ? launch_generic_t<2>(pl, l, weights[k], sketch, st, kap_max)
                                            : launch_generic_t<4>(pl, l, weights[k], sketch, st, kap_max);
      if (s != USK_OK) return s;
    }
  }
  usk_status s = USK_OK;
  for (int upl : {4, 2, 1}) {
    if (!grp[upl].empty() && s == USK_OK) s = launch_fast(pl, upl, grp[upl], sketch, st, kap_max);
    if (!ggrp[upl].empty() && s == USK_OK) s = launch_fast(pl, upl, ggrp[upl], sketch, st, kap_max, nullptr, true);
  }
  // output-row units (L31): transpose batches of layers (<= 64 MB, or one layer) into a stream-ordered
  // scratch buffer and build them as input-dim units of W^T; stream order serialises the batches
  const int es = pl->cell_bytes();
  const size_t cap = (size_t)64 << 20;
  for (int upl : {4, 2, 1}) {
    auto& tg = tgrp[upl];
    for (size_t a = 0; a < tg.size() && s == USK_OK;) {
      size_t b = a, bytes = 0;
      while (b < tg.size()) {
        const LayerGeom& L = pl->layers[tg[b].first];
        const size_t lb = ((size_t)(L.out * L.in * es) + 255) / 256 * 256;
        if (b > a && bytes + lb > cap) break;
        bytes += lb;
        ++b;
      }
      char* wt = nullptr;
      USK_CUDA(cudaMallocAsync(&wt, bytes, st));
      std::vector<std::pair<int32_t, const void*>> batch;
      size_t off = 0;
      for (size_t k = a; k < b; ++k) {
        const LayerGeom& L = pl->layers[tg[k].first];
        const dim3 grid((unsigned)((L.in + 31) / 32), (unsigned)((L.out + 31) / 32));
        if (es == 2) k_transpose<2><<<grid, dim3(32, 8), 0, st>>>(tg[k].second, wt + off, L.out, L.in, L.out);
        else k_transpose<4><<<grid, dim3(32, 8), 0, st>>>(tg[k].second, wt + off, L.out, L.in, L.out);
        USK_LAUNCHED("k_transpose");
        batch.push_back({tg[k].first, wt + off});
        off += ((size_t)(L.out * L.in * es) + 255) / 256 * 256;
      }
      s = launch_fast(pl, upl, batch, sketch, st, kap_max);
      cudaError_t e = cudaFreeAsync(wt, st);
      if (s == USK_OK && e != cudaSuccess) s = cuda_fail(e, "usk_build: cudaFreeAsync");
      a = b;
    }
  }
  return s;
}

// Quantised plans (L25): raw states are built into a stream-ordered temporary buffer
// with the plan's (G-aligned) cell offsets, then quantised group by group into the sketch:
// codes at byte 0, fp32 scales at scales_off.  Groups never straddle layers, so a layer-sharded
// build quantises exactly the groups of its layers.
// Top-K plans (L29): per built layer, a device top-K selection (CUB radix sort of the
// selection keys) writes the side table, and a copy of W with the outliers set to +Inf (a key no
// finite weight loses to, so they never enter a cell) is sketched instead of W.
static usk_status launch_build_topk(const usk_plan* pl, const void* const* weights, const int32_t* layer_ids,
                                    int32_t n, void* sketch, cudaStream_t st) {
  const int es = pl->cell_bytes();
  std::vector<void*> temps;
  std::vector<const void*> wb(n);
  usk_status s = USK_OK;
  auto cuda_ok = [&](cudaError_t e, const char* what) {
    if (e != cudaSuccess && s == USK_OK) s = cuda_fail(e, what);
    return s == USK_OK;
  };
  for (int32_t k = 0; k < n && s == USK_OK; ++k) {
    const LayerGeom& L = pl->layers[layer_ids ? layer_ids[k] : k];
    const int64_t ne = L.out * L.in, K = L.n_out;
    wb[k] = weights[k];
    if (K == 0) continue;
    void *Wc = nullptr, *keys = nullptr, *keys2 = nullptr, *idx = nullptr, *idx2 = nullptr, *tmp = nullptr;
    size_t tb1 = 0, tb2 = 0;
    if (!cuda_ok(cudaMallocAsync(&Wc, (size_t)ne * es, st), "cudaMallocAsync")) break;
    temps.push_back(Wc);
    cuda_ok(cudaMemcpyAsync(Wc, weights[k], (size_t)ne * es, cudaMemcpyDeviceToDevice, st), "cudaMemcpyAsync");
    cuda_ok(cudaMallocAsync(&keys, (size_t)ne * 8, st), "cudaMallocAsync");
    cuda_ok(cudaMallocAsync(&keys2, (size_t)ne * 8, st), "cudaMallocAsync");
    cuda_ok(cudaMallocAsync(&idx, (size_t)K * 4, st), "cudaMallocAsync");
    cuda_ok(cudaMallocAsync(&idx2, (size_t)K * 4, st), "cudaMallocAsync");
    cuda_ok(cub::DeviceRadixSort::SortKeysDescending(nullptr, tb1, (unsigned long long*)keys,
                                                     (unsigned long long*)keys2, (int)ne, 0, 64, st), "cub");
    cuda_ok(cub::DeviceRadixSort::SortKeys(nullptr, tb2, (uint32_t*)idx, (uint32_t*)idx2, (int)K, 0, 32, st), "cub");
    cuda_ok(cudaMallocAsync(&tmp, std::max(tb1, tb2), st), "cudaMallocAsync");
    if (s != USK_OK) break;
    k_topk_keys<<<(unsigned)((ne + 255) / 256), 256, 0, st>>>(weights[k], es, ne, (unsigned long long*)keys,
                                                             pl->d_err);
    cuda_ok(cudaGetLastError(), "k_topk_keys");
    count_launch();
    cuda_ok(cub::DeviceRadixSort::SortKeysDescending(tmp, tb1, (unsigned long long*)keys, (unsigned long long*)keys2,
                                                     (int)ne, 0, 64, st), "cub sort");
    count_launch();
    k_topk_take<<<(unsigned)((K + 255) / 256), 256, 0, st>>>((unsigned long long*)keys2, K, (uint32_t*)idx);
    cuda_ok(cudaGetLastError(), "k_topk_take");
    count_launch();
    cuda_ok(cub::DeviceRadixSort::SortKeys(tmp, tb2, (uint32_t*)idx, (uint32_t*)idx2, (int)K, 0, 32, st), "cub sort");
    count_launch();
    char* tab = reinterpret_cast<char*>(sketch) + L.out_off;
    k_topk_finish<<<(unsigned)((K + 255) / 256), 256, 0, st>>>((uint32_t*)idx2, K, weights[k], es,
                                                               reinterpret_cast<int32_t*>(tab),
                                                               tab + (K * 4 + 15) / 16 * 16, Wc);
    cuda_ok(cudaGetLastError(), "k_topk_finish");
    count_launch();
    void* frees[] = {keys, keys2, idx, idx2, tmp};
    for (void* f : frees) cuda_ok(cudaFreeAsync(f, st), "cudaFreeAsync");
    wb[k] = Wc;
  }
  if (s == USK_OK) s = launch_build_raw(pl, wb.data(), layer_ids, n, sketch, st, 0xFF000000u);
  for (void* t : temps) cudaFreeAsync(t, st);
  return s;
}

// query layout (usk.h USK_LAYOUT_QUERY): K2 writes the rho16 chunk slices directly when every requested
// layer takes the fast build (else packed.cu builds unit-major cells into scratch and packs them)
bool build_qfast_ok(const usk_plan* pl, const int32_t* layer_ids, int32_t n) {
  if (pl->dtype != USK_BF16 || pl->gran != USK_GRAN_ROW || pl->q || pl->topk) return false;
  for (int32_t k = 0; k < n; ++k) {
    const int32_t l = layer_ids ? layer_ids[k] : k;
    if (!fast_upl(pl, l)) return false;
    // the fused write-out fills whole slices of identity-ordered chunks of >= 128 units and all rows,
    // or (table-driven, class-ordered layers, ledger L34) each key group's slices of its own chunk
    const LayerGeom& L = pl->layers[l];
    if (L.qperm) continue;  // table-driven write-out (per key group: chunk, slot, rows from the plan)
    if (L.qmixed || L.qcw < 128) return false;
    for (int c = 0; c < L.qchunks; ++c)
      if (pl->h_qc_M[L.qchunk0 + c] != pl->M) return false;
  }
  return true;
}

usk_status launch_build_qfast(const usk_plan* pl, const void* const* weights, const int32_t* layer_ids, int32_t n,
                              void* qsketch, cudaStream_t st) {
  std::vector<std::pair<int32_t, const void*>> grp[5], ggrp[5];
  for (int32_t k = 0; k < n; ++k) {
    const int32_t l = layer_ids ? layer_ids[k] : k;
    (layer_gk_ok(pl, l) ? ggrp : grp)[fast_upl(pl, l)].push_back({l, weights[k]});
  }
  for (int upl : {4, 2, 1}) {
    usk_status s = USK_OK;
    if (!grp[upl].empty()) s = launch_fast(pl, upl, grp[upl], nullptr, st, 0xFEFFFFFFu, qsketch);
    if (s == USK_OK && !ggrp[upl].empty()) s = launch_fast(pl, upl, ggrp[upl], nullptr, st, 0xFEFFFFFFu, qsketch, true);
    if (s != USK_OK) return s;
  }
  return USK_OK;
}

usk_status launch_build_rows(const usk_plan* pl, int32_t l, int64_t r0, int64_t r1, const void* w_rows, void* sketch,
                             cudaStream_t st) {
  const int upl = fast_upl(pl, l, true);
  if (!upl) return fail(USK_EUNSUPPORTED, "usk_build_rows: layer not eligible for the fast build");
  const LayerGeom& L = pl->layers[l];
  const int es = pl->cell_bytes();
  const int64_t rows = r1 - r0;
  const int64_t ld = (rows * es + 15) / 16 * 16 / es;  // W^T row pitch: 16-B multiple for the tensor map
  char* wt = nullptr;
  USK_CUDA(cudaMallocAsync(&wt, (size_t)(L.in * ld * es), st));
  const dim3 grid((unsigned)((L.in + 31) / 32), (unsigned)((rows + 31) / 32));
  if (es == 2) k_transpose<2><<<grid, dim3(32, 8), 0, st>>>(w_rows, wt, rows, L.in, ld);
  else k_transpose<4><<<grid, dim3(32, 8), 0, st>>>(w_rows, wt, rows, L.in, ld);
  USK_LAUNCHED("k_transpose");
  // one task: W^T [in, rows] -- its columns are the units unit_begin + r0 .. unit_begin + r1 - 1
  BuildArgs A{};
  A.M = pl->M;
  A.hc = pl->hc;
  A.ncols = pl->d_ncols;
  A.nrows = pl->d_nrows;
  A.offsets = pl->d_offsets;
  A.ukeys = pl->d_keys;
  A.R4 = pl->d_R4;
  A.sketch = sketch;
  A.err = pl->d_err;
  A.kap_max = 0xFEFFFFFFu;
  A.maxMN = std::max(1, pl->M * L.max_ncols);
  const int TJ = 32 * upl;
  BuildTask& t = A.task[A.n_tasks++];
  t.W = wt;
  t.out = L.in;
  t.in = rows;
  t.unit_base = L.unit_begin + r0;
  t.tile_begin = 0;
  usk_status s = USK_OK;
  if (!make_w_map(&t.map, wt, L.in, rows, es, TJ, ld)) s = fail(USK_ECUDA, "usk_build_rows: cuTensorMapEncodeTiled failed");
  const int tiles = (int)((rows + TJ - 1) / TJ);
  if (s == USK_OK) {
    if (pl->dtype == USK_BF16)
      s = upl == 4 ? launch_fast_m<uint16_t, 4>(A, tiles, pl->hash, st)
          : upl == 2 ? launch_fast_m<uint16_t, 2>(A, tiles, pl->hash, st) : launch_fast_m<uint16_t, 1>(A, tiles, pl->hash, st);
    else
      s = upl == 4 ? launch_fast_m<uint32_t, 4>(A, tiles, pl->hash, st)
          : upl == 2 ? launch_fast_m<uint32_t, 2>(A, tiles, pl->hash, st) : launch_fast_m<uint32_t, 1>(A, tiles, pl->hash, st);
  }
  cudaError_t e = cudaFreeAsync(wt, st);
  if (s == USK_OK && e != cudaSuccess) s = cuda_fail(e, "usk_build_rows: cudaFreeAsync");
  return s;
}

usk_status launch_build(const usk_plan* pl, const void* const* weights, const int32_t* layer_ids, int32_t n,
                        void* sketch, cudaStream_t st) {
  if (pl->topk) return launch_build_topk(pl, weights, layer_ids, n, sketch, st);
  if (!pl->q) return launch_build_raw(pl, weights, layer_ids, n, sketch, st);
  const int es = pl->cell_bytes();
  void* raw = nullptr;
  USK_CUDA(cudaMallocAsync(&raw, (size_t)pl->total_cells * es + 256, st));
  const unsigned fb = (unsigned)((pl->total_cells + 255) / 256);
  if (es == 2) k_fill_inf<2><<<fb, 256, 0, st>>>(raw, pl->total_cells);
  else k_fill_inf<4><<<fb, 256, 0, st>>>(raw, pl->total_cells);
  USK_LAUNCHED("k_fill_inf");
  usk_status s = launch_build_raw(pl, weights, layer_ids, n, raw, st);
  uint8_t* codes = reinterpret_cast<uint8_t*>(sketch);
  float* scales = reinterpret_cast<float*>(reinterpret_cast<char*>(sketch) + pl->scales_off);
  for (int32_t k = 0; k < n && s == USK_OK; ++k) {
    const LayerGeom& L = pl->layers[layer_ids ? layer_ids[k] : k];
    const int64_t g0 = L.cell_begin / pl->G, g1 = (L.cell_begin + L.n_cells + pl->G - 1) / pl->G;
    if (g1 <= g0) continue;
    const unsigned blocks = (unsigned)((g1 - g0 + 7) / 8);  // 8 warps (groups) per block
    if (es == 2) {
      if (pl->q == 4) k_quantize<2, 4><<<blocks, 256, 0, st>>>(raw, g0, g1, pl->G, codes, scales);
      else k_quantize<2, 8><<<blocks, 256, 0, st>>>(raw, g0, g1, pl->G, codes, scales);
    } else {
      if (pl->q == 4) k_quantize<4, 4><<<blocks, 256, 0, st>>>(raw, g0, g1, pl->G, codes, scales);
      else k_quantize<4, 8><<<blocks, 256, 0, st>>>(raw, g0, g1, pl->G, codes, scales);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) s = cuda_fail(e, "k_quantize");
    else count_launch();
  }
  cudaError_t e = cudaFreeAsync(raw, st);
  if (s == USK_OK && e != cudaSuccess) s = cuda_fail(e, "usk_build: cudaFreeAsync");
  return s;
}

}  // namespace usk
