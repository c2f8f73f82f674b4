// query.cu -- K3 reconstruct, K4 sketch-GEMV (decode), K6 importance.
//
// Query of one weight (Eq. 3 + Eq. 5; §3.1 "hash ... retrieved by the above
// indices in a batch ... interpreting these intermediate results"):
//   w'(o, j) = the bonded cell of maximum |.| over rows i < M (ties -> non-negative, L1/L2).
//
// Fast path (ROW granularity, one input dimension per unit).
//   * Each CTA owns one CHUNK of TJ = 32*UPL consecutive units (input dims) of one layer and a
//     contiguous range of 32-row SUBTILES; the chunk's cells are staged into shared memory once
//     and reused over the whole row range (a cell is hit by ~out/N rows, so a CTA must cover
//     many rows for the staging to amortise).  Grid = sum over layers of n_chunks x cpc, with
//     cpc (CTAs per chunk) chosen so that the grid is one resident wave.
//   * Lane L owns units UPL*L+v.  Their cells sit in shared memory as rho codes
//         rho = rotl(bits_hi, 1) ^ 1 = (mag << 1) | (1 - sign)
//     at byte address  cells + 4*(v*32*maxMN + k*32 + L)  -- always bank L, so the M random
//     gathers of a warp never conflict.  The Eq. 5 select is an integer max (VIMNMX3 for M=3)
//     and rotr(rho, 1) is the IEEE pattern of -w', so the GEMV multiplies by -x (exact).
//     Per weight and lane: 1 LOP3 (R(o) ^ K_u) + M x (IMAD, IMAD.HI, LEA, LDS) + max + SHF + FFMA.
//   * Missing units of a ragged chunk point at a shared "zero" cell (rho of +0) with x = 0, so
//     the inner loop has no branches.  R(o) for a subtile is one register per lane (lane r holds
//     R(o0 + r)), broadcast with SHFL, prefetched one subtile ahead.
//   * GEMV: per subtile a warp holds 32 row partials per lane; a transpose butterfly leaves row r
//     on lane r.  Partials go to a row-major [rows][CP] workspace; the warp that completes a
//     subtile's last chunk (atomic counter per subtile) sums the chunks in fixed order with
//     float4 loads (deterministic, no float atomics) and writes y.
//   * Programmatic dependent launch: the chunk is staged (sketch only) before
//     griddepcontrol.wait, overlapping the previous kernel; x is read after it.
//     usk_linear_batch puts several linears that share x (q|k|v, gate|up) in one launch.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "common.cuh"
#include "ptx.cuh"

namespace usk {
namespace {

#ifndef USK_QUERY_THREADS
#define USK_QUERY_THREADS 512
#endif
constexpr int kQThreads = USK_QUERY_THREADS;
constexpr int kMaxBatch = 8;
constexpr int kSubRows = 16;  // rows per warp work item (subtile)
constexpr int kCellsWordOffset = 32 + 160;  // zero cells + chunk unit offsets (<= 129)

extern __shared__ __align__(16) uint32_t qsm[];  // dynamic shared memory of the query kernels

// 32-bit shared load at a byte offset from qsm: compiles to LDS [R + UR] (base folded), and as
// an ordinary load it can be scheduled freely around the address arithmetic.
__device__ __forceinline__ uint32_t lds32(uint32_t off) {
  return *reinterpret_cast<const uint32_t*>(reinterpret_cast<const char*>(qsm) + off);
}

struct QLayer {
  int64_t unit_base;   // global unit id of the layer's first unit
  int64_t o_begin;     // first output row
  int64_t rows;        // rows in [o_begin, o_end)
  int32_t n_chunks;    // unit chunks of TJ
  int32_t n_sub;       // 16-row subtiles
  int32_t cpc;         // GEMV: CTAs per chunk; reconstruct: CTAs of the layer
  int32_t cta_begin;   // first CTA of this layer in the launch
  int32_t CP;          // row stride of the partial workspace (>= n_chunks, multiple of 4)
  int32_t pad;
  // gemv
  void* y;
  float* partial;      // [rows][CP]
  uint32_t* counters;  // [n_sub] split-K completion counts
  uint32_t* work;      // [2 * n_chunks]: per chunk, next subtile to grab and warps finished
  // reconstruct
  void* w_out;
  int64_t ld_out;
};

struct QArgs {
  QLayer layer[kMaxBatch];
  int32_t n_layers;
  int32_t M;
  int32_t maxMN;       // smem slot stride (cells) = max over the launch's layers
  int32_t early_trigger;
  int64_t in;          // in_features (shared by the batch)
  const void* sketch;
  const int32_t* ncols;
  const int64_t* offsets;
  const uint32_t* ukeys;
  const uint32_t* R;
  HashConsts hc;
  const void* x;
  int32_t x_bf16;
  int32_t y_bf16;
  unsigned long long* timeline;  // debug only (USK_TIMELINE=1): 4 globaltimer stamps per CTA
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

template <int UPL, int MT>
struct LaneState {
  static constexpr int MR = MT > 0 ? MT : 1;
  uint32_t K[UPL], N[UPL];
  uint32_t rb[UPL][MR];  // shared byte address of (unit v, sketch row i, column 0) for this lane
  uint32_t rstride[UPL]; // bytes between sketch rows (runtime-M kernels)
};

// Stage one chunk's cells (rho codes, bank-private layout) and set up the lane state.
template <typename E, int UPL, int MT>
__device__ __forceinline__ void stage_chunk(const QArgs& A, const QLayer& Ly, int64_t j0, int nu, uint32_t* cells,
                                            uint32_t* zero, LaneState<UPL, MT>& S) {
  constexpr int TJ = 32 * UPL;
  constexpr int ES = sizeof(E);
  const int lane = threadIdx.x & 31;
  // The chunk's units are consecutive in the sketch, so their cells are one contiguous byte range:
  // a single TMA bulk copy (cp.async.bulk, mbarrier completion) brings it into a raw shared
  // buffer; threads then convert shared -> shared into the bank-private rho layout.
  uint64_t* bar = reinterpret_cast<uint64_t*>(zero + 32);
  uint32_t* s_shift = zero + 34;
  unsigned char* raw = reinterpret_cast<unsigned char*>(cells + UPL * 32 * A.maxMN);
  const int64_t ubase = Ly.unit_base + j0;
  if (threadIdx.x == 0) {
    const uint64_t g0 = (uint64_t)A.offsets[ubase] * ES, g1 = (uint64_t)A.offsets[ubase + nu] * ES;
    const uint64_t a0 = g0 & ~uint64_t(15), a1 = (g1 + 15) & ~uint64_t(15);
    mbar_init(bar, 1);
    fence_mbar_init();
    mbar_arrive_expect_tx(bar, (uint32_t)(a1 - a0));
    bulk_g2s(raw, reinterpret_cast<const unsigned char*>(A.sketch) + a0, (uint32_t)(a1 - a0), bar);
    *s_shift = (uint32_t)(g0 - a0);
  }
  const int ul = threadIdx.x % TJ;
  int64_t u_off = 0;
  int mn = 0;
  if (ul < nu) {  // overlaps the copy
    u_off = A.offsets[ubase + ul] - A.offsets[ubase];
    mn = A.M * A.ncols[ubase + ul];
  }
  if (threadIdx.x < 32) zero[threadIdx.x] = 1u;  // rho(+0)
  __syncthreads();                                 // barrier init + shift visible
  mbar_wait(bar, 0);
  {
    const unsigned char* src = raw + *s_shift + u_off * ES;
    uint32_t* dst = cells + (ul % UPL) * 32 * A.maxMN + ul / UPL;
    constexpr int KS = kQThreads / TJ;
#pragma unroll 4
    for (int k = threadIdx.x / TJ; k < mn; k += KS) {
      const uint32_t b = ES == 2 ? ((uint32_t)reinterpret_cast<const uint16_t*>(src)[k] << 16)
                                 : reinterpret_cast<const uint32_t*>(src)[k];
      dst[k * 32] = rotl1(b) ^ 1u;
    }
  }
  const uint32_t cbase = (uint32_t)((cells - qsm) * 4), zbase = (uint32_t)((zero - qsm) * 4);  // byte offsets
#pragma unroll
  for (int v = 0; v < UPL; ++v) {
    const int ul = UPL * lane + v;
    if (ul < nu) {
      const int64_t u = Ly.unit_base + j0 + ul;
      S.K[v] = A.ukeys[u];
      S.N[v] = (uint32_t)A.ncols[u];
      const uint32_t b0 = cbase + 4u * (uint32_t)(v * 32 * A.maxMN + lane);
      S.rstride[v] = S.N[v] * 128u;
#pragma unroll
      for (int i = 0; i < LaneState<UPL, MT>::MR; ++i) S.rb[v][i] = b0 + (uint32_t)i * S.rstride[v];
    } else {
      S.K[v] = 0;
      S.N[v] = 1;  // idx is always 0
      S.rstride[v] = 0;
#pragma unroll
      for (int i = 0; i < LaneState<UPL, MT>::MR; ++i) S.rb[v][i] = zbase + 4u * lane;
    }
  }
}

// rho code of w'(o, unit v) for this lane
template <int UPL, int MT, int HASH>
__device__ __forceinline__ uint32_t select_rho(const QArgs& A, const LaneState<UPL, MT>& S, int v, uint32_t Rv,
                                               int64_t o) {
  const uint32_t h = Rv ^ S.K[v];
  if constexpr (MT > 0 && HASH == USK_HASH_X) {
    uint32_t m[MT];
#pragma unroll
    for (int i = 0; i < MT; ++i) m[i] = lds32(S.rb[v][i] + (__umulhi(h * A.hc.a[i], S.N[v]) << 7));
    uint32_t best = m[0];
#pragma unroll
    for (int i = 1; i < MT; ++i) best = max(best, m[i]);
    return best;
  } else {
    uint32_t best = 0, base = S.rb[v][0];
    for (int i = 0; i < A.M; ++i) {
      const uint32_t idx = (HASH == USK_HASH_X) ? __umulhi(h * A.hc.a[i], S.N[v]) : (uint32_t)(o % S.N[v]);
      best = max(best, lds32(base + (idx << 7)));
      base += S.rstride[v];
    }
    return best;
  }
}

// Row r of the warp's 16 partial rows ends on lanes r and r + 16 (fixed-order butterfly: 4
// exchange-and-halve stages inside each half-warp, then the two halves are added).
__device__ __forceinline__ float transpose_reduce16(float (&acc)[16], int lane) {
#pragma unroll
  for (int m = 8; m >= 1; m >>= 1) {
    const bool up = (lane & m) != 0;
#pragma unroll
    for (int i = 0; i < m; ++i) {
      const float send = up ? acc[i] : acc[i + m];
      const float keep = up ? acc[i + m] : acc[i];
      acc[i] = keep + __shfl_xor_sync(0xffffffffu, send, m);
    }
  }
  return acc[0] + __shfl_xor_sync(0xffffffffu, acc[0], 16);
}

// y[r] = sum over chunks (fixed order) of the row-major partials; float4 loads, all issued up front.
__device__ __forceinline__ void reduce_row(const QArgs& A, const QLayer& Ly, int64_t r) {
  const float4* p = reinterpret_cast<const float4*>(Ly.partial + r * Ly.CP);
  float t = 0.f;
  int c = 0;
  for (; c + 32 <= Ly.n_chunks; c += 32) {
    float4 q[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) q[k] = __ldcg(p + c / 4 + k);
#pragma unroll
    for (int k = 0; k < 8; ++k) t = t + q[k].x + q[k].y + q[k].z + q[k].w;
  }
  for (; c < Ly.n_chunks; c += 4) {
    const float4 q = __ldcg(p + c / 4);
    const float w4[4] = {q.x, q.y, q.z, q.w};
    for (int k = 0; k < 4 && c + k < Ly.n_chunks; ++k) t += w4[k];
  }
  if (A.y_bf16) {
    const uint32_t bb = __float_as_uint(t);
    reinterpret_cast<uint16_t*>(Ly.y)[r] = (uint16_t)((bb + 0x7FFFu + ((bb >> 16) & 1u)) >> 16);
  } else {
    reinterpret_cast<float*>(Ly.y)[r] = t;
  }
}

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

#ifndef USK_QUERY_MINB
#define USK_QUERY_MINB 2
#endif

template <typename E, int UPL, int MT, int HASH, bool GEMV>
__global__ void __launch_bounds__(kQThreads, USK_QUERY_MINB) k_query_fast(const __grid_constant__ QArgs A) {
  constexpr int TJ = 32 * UPL;
  uint32_t* zero = qsm;
  uint32_t* cells = qsm + kCellsWordOffset;  // [zero: 32 words][unit offsets: 160][cells]
  __shared__ int s_next;  // next subtile of this CTA's range (warps grab dynamically)
  __shared__ int s_last;
  const int lane = threadIdx.x & 31;

  int li = 0;
  while (li + 1 < A.n_layers && A.layer[li + 1].cta_begin <= (int)blockIdx.x) ++li;
  const QLayer& Ly = A.layer[li];
  const int b = blockIdx.x - Ly.cta_begin;
  int chunk, part = 0, sub0 = 0, sub1 = 0;
  if constexpr (GEMV) {
    // cpc CTAs per chunk; every chunk uses the same row partition (part q covers subtiles
    // [q n_sub / cpc, (q+1) n_sub / cpc)), so one counter per part collects the chunks
    chunk = b / Ly.cpc;
    part = b % Ly.cpc;
    sub0 = (int)(((int64_t)part * Ly.n_sub) / Ly.cpc);
    sub1 = (int)(((int64_t)(part + 1) * Ly.n_sub) / Ly.cpc);
  } else {
    // the layer's cpc CTAs are spread over its chunks as evenly as possible; each chunk's CTAs
    // split its subtiles evenly (static)
    chunk = (int)(((int64_t)b * Ly.n_chunks) / Ly.cpc);
    const int first = (int)(((int64_t)chunk * Ly.cpc + Ly.n_chunks - 1) / Ly.n_chunks);
    const int nparts = (int)((((int64_t)(chunk + 1) * Ly.cpc + Ly.n_chunks - 1) / Ly.n_chunks) - first);
    part = b - first;
    sub0 = (int)(((int64_t)part * Ly.n_sub) / nparts);
    sub1 = (int)(((int64_t)(part + 1) * Ly.n_sub) / nparts);
  }
  const int64_t j0 = (int64_t)chunk * TJ;
  const int nu = (int)min((int64_t)TJ, A.in - j0);

  if (A.timeline && threadIdx.x == 0) A.timeline[blockIdx.x * 4 + 0] = gtimer();
  LaneState<UPL, MT> S;
  stage_chunk<E, UPL, MT>(A, Ly, j0, nu, cells, zero, S);
  float nx[UPL];
  if constexpr (GEMV) {
    pdl_wait();  // x may be written by the previous kernel on the stream
    if (A.early_trigger) pdl_trigger();
#pragma unroll
    for (int v = 0; v < UPL; ++v) {
      const int64_t j = j0 + UPL * lane + v;
      float xv = 0.f;
      if (UPL * lane + v < nu)
        xv = A.x_bf16 ? __uint_as_float((uint32_t)reinterpret_cast<const uint16_t*>(A.x)[j] << 16)
                      : reinterpret_cast<const float*>(A.x)[j];
      nx[v] = -xv;  // rotr(rho) decodes to -w'
    }
  }
  if (threadIdx.x == 0) s_next = sub0 + 0;
  __syncthreads();
  if (A.timeline && threadIdx.x == 0) A.timeline[blockIdx.x * 4 + 1] = gtimer();

  const int rl = lane & (kSubRows - 1);  // lanes r and r + 16 both hold R(o0 + r)
  auto next_sub = [&]() -> int {
    int g = 0;
    if (lane == 0) g = atomicAdd(&s_next, 1);
    return __shfl_sync(0xffffffffu, g, 0);
  };
  const int sub_end = sub1;
  int sub = next_sub();
  uint32_t Rl = 0;
  // R(o) = fmix32(o ^ rho): lane r computes its own row's mix (6 integer ops per subtile and
  // lane, no memory access); SHFL broadcasts it row by row
  if (sub < sub_end) Rl = fmix32((uint32_t)(Ly.o_begin + min((int64_t)sub * kSubRows + rl, Ly.rows - 1)) ^ A.hc.rho);
  while (sub < sub_end) {
    const int nxt = next_sub();  // issued now, consumed after this subtile's math
    const int64_t r0 = (int64_t)sub * kSubRows;  // first local row of the subtile
    const int nrow = (int)min((int64_t)kSubRows, Ly.rows - r0);
    if constexpr (GEMV) {
      float acc[kSubRows];
#pragma unroll
      for (int r = 0; r < kSubRows; ++r) {
        const uint32_t Rv = __shfl_sync(0xffffffffu, Rl, r);
        float a = 0.f;
#pragma unroll
        for (int v = 0; v < UPL; ++v)
          a = fmaf(nx[v], __uint_as_float(rotr1(select_rho<UPL, MT, HASH>(A, S, v, Rv, Ly.o_begin + r0 + r))), a);
        acc[r] = a;
      }
      const float s = transpose_reduce16(acc, lane);
      if (lane < nrow) Ly.partial[(r0 + lane) * Ly.CP + chunk] = s;
    } else {
      const bool full_tile = (nu == TJ);
      E* dst = reinterpret_cast<E*>(Ly.w_out) + r0 * Ly.ld_out + j0 + UPL * lane;
#pragma unroll 4
      for (int r = 0; r < kSubRows; ++r, dst += Ly.ld_out) {
        const uint32_t Rv = __shfl_sync(0xffffffffu, Rl, r);
        if (r >= nrow) continue;
        uint32_t wb[UPL];
#pragma unroll
        for (int v = 0; v < UPL; ++v)
          wb[v] = rotr1(select_rho<UPL, MT, HASH>(A, S, v, Rv, Ly.o_begin + r0 + r)) ^ 0x80000000u;
        if constexpr (sizeof(E) == 2) {
          if (full_tile) {
            if constexpr (UPL == 4) {
              *reinterpret_cast<uint2*>(dst) = make_uint2(__byte_perm(wb[0], wb[1 % UPL], 0x7632),
                                                          __byte_perm(wb[2 % UPL], wb[3 % UPL], 0x7632));
            } else if constexpr (UPL == 2) {
              *reinterpret_cast<uint32_t*>(dst) = __byte_perm(wb[0], wb[1 % UPL], 0x7632);
            } else {
              dst[0] = (E)(wb[0] >> 16);
            }
          } else {
#pragma unroll
            for (int v = 0; v < UPL; ++v)
              if (UPL * lane + v < nu) dst[v] = (E)(wb[v] >> 16);
          }
        } else {
          if (full_tile && UPL == 4) {
            *reinterpret_cast<uint4*>(dst) = make_uint4(wb[0], wb[1 % UPL], wb[2 % UPL], wb[3 % UPL]);
          } else if (full_tile && UPL == 2) {
            *reinterpret_cast<uint2*>(dst) = make_uint2(wb[0], wb[1 % UPL]);
          } else {
#pragma unroll
            for (int v = 0; v < UPL; ++v)
              if (UPL * lane + v < nu) dst[v] = wb[v];
          }
        }
      }
    }
    sub = nxt;
    if (sub < sub_end) Rl = fmix32((uint32_t)(Ly.o_begin + min((int64_t)sub * kSubRows + rl, Ly.rows - 1)) ^ A.hc.rho);
  }
  if (A.timeline && lane == 0) atomicMax(&A.timeline[blockIdx.x * 4 + 2], gtimer());
  if constexpr (GEMV) {
    // ---- split-K: one release per CTA; the CTA that completes row part `part` (the n_chunks-th
    // arrival) sums its rows' chunk partials in fixed chunk order and writes y
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = (atomicAdd(&Ly.counters[part], 1u) == (uint32_t)Ly.n_chunks - 1);
    __syncthreads();
    if (!A.early_trigger) pdl_trigger();
    if (s_last) {
      __threadfence();
      const int64_t ra = (int64_t)sub0 * kSubRows, rb = min((int64_t)sub1 * kSubRows, Ly.rows);
      for (int64_t r = ra + threadIdx.x; r < rb; r += kQThreads) reduce_row(A, Ly, r);
      if (threadIdx.x == 0) Ly.counters[part] = 0u;  // leave the workspace zeroed for the next call
    }
  }
  if (A.timeline && lane == 0) atomicMax(&A.timeline[blockIdx.x * 4 + 3], gtimer());
}

// ------------------------------------------------------------------ generic query path
struct GenQ {
  const void* sketch;
  const int32_t* ncols;
  const int64_t* offsets;
  const uint32_t* ukeys;
  HashConsts hc;
  int64_t unit_base, out, in;
  int32_t M, gran, g, hash, es;
};

__device__ __forceinline__ uint32_t gen_weight_bits_hi(const GenQ& Q, int64_t o, int64_t j) {
  int64_t t, p;
  if (Q.gran == USK_GRAN_ROW) { t = j / Q.g; p = (j - t * Q.g) * Q.out + o; }
  else { t = 0; p = j * Q.out + o; }
  const int64_t u = Q.unit_base + t;
  const uint32_t N = (uint32_t)Q.ncols[u];
  const int64_t off = Q.offsets[u];
  const uint32_t h = fmix32((uint32_t)p ^ Q.hc.rho) ^ Q.ukeys[u];
  uint32_t best = 0;
  for (int i = 0; i < Q.M; ++i) {
    const uint32_t idx = Q.hash == USK_HASH_X ? __umulhi(h * Q.hc.a[i], N) : (uint32_t)(p % N);
    const int64_t c = off + (int64_t)i * N + idx;
    uint32_t b = Q.es == 2 ? ((uint32_t)reinterpret_cast<const uint16_t*>(Q.sketch)[c] << 16)
                           : reinterpret_cast<const uint32_t*>(Q.sketch)[c];
    best = max(best, rotl1(b) ^ 1u);
  }
  return rotr1(best) ^ 0x80000000u;
}

__global__ void k_reconstruct_gen(GenQ Q, int64_t o0, int64_t o1, void* w_out, int64_t ld) {
  const int64_t n = (o1 - o0) * Q.in;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / Q.in, j = e - r * Q.in;
    const uint32_t b = gen_weight_bits_hi(Q, o0 + r, j);
    if (Q.es == 2) reinterpret_cast<uint16_t*>(w_out)[r * ld + j] = (uint16_t)(b >> 16);
    else reinterpret_cast<uint32_t*>(w_out)[r * ld + j] = b;
  }
}

// one warp per output row, lanes over j, fixed-order warp reduction
__global__ void k_gemv_gen(GenQ Q, int64_t o0, int64_t o1, const void* x, int32_t x_bf16, void* y, int32_t y_bf16) {
  const int64_t r = blockIdx.x * (int64_t)(blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (o0 + r >= o1) return;
  float s = 0.f;
  for (int64_t j = lane; j < Q.in; j += 32) {
    const float w = __uint_as_float(gen_weight_bits_hi(Q, o0 + r, j));
    const float xv = x_bf16 ? __uint_as_float((uint32_t)reinterpret_cast<const uint16_t*>(x)[j] << 16)
                            : reinterpret_cast<const float*>(x)[j];
    s = fmaf(xv, w, s);
  }
  for (int m = 16; m >= 1; m >>= 1) s += __shfl_xor_sync(0xffffffffu, s, m);
  if (lane == 0) {
    if (y_bf16) {
      const uint32_t b = __float_as_uint(s);
      reinterpret_cast<uint16_t*>(y)[r] = (uint16_t)((b + 0x7FFFu + ((b >> 16) & 1u)) >> 16);
    } else {
      reinterpret_cast<float*>(y)[r] = s;
    }
  }
}

// ------------------------------------------------------------------ K6: importance (Eq. 7)
__global__ void k_importance(const void* A, int32_t bf16, int64_t N, int64_t d, float* I) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= d) return;
  double s = 0.0;
  for (int64_t k = 0; k < N; ++k) {
    const double a = bf16 ? (double)__uint_as_float((uint32_t)reinterpret_cast<const uint16_t*>(A)[k * d + j] << 16)
                          : (double)reinterpret_cast<const float*>(A)[k * d + j];
    s += a * a;
  }
  I[j] = (float)(s / (double)N);
}

// ------------------------------------------------------------------ host side
bool fast_eligible(const usk_plan* pl) { return pl->gran == USK_GRAN_ROW && pl->g == 1; }

constexpr size_t kSmemMax = 220 * 1024;

// [zero + mbarrier + unit slots][rho cells][raw chunk bytes of the bulk copy (+ alignment slack)]
size_t smem_bytes(int upl, int maxMN, int es) {
  return kCellsWordOffset * 4 + (size_t)32 * upl * maxMN * 4 + (size_t)32 * upl * maxMN * es + 48;
}

template <typename E, int UPL, bool GEMV>
void* pick_m(int M, int hash) {
  if (hash == USK_HASH_IDENTITY) return (void*)k_query_fast<E, UPL, 0, USK_HASH_IDENTITY, GEMV>;
  switch (M) {
    case 1: return (void*)k_query_fast<E, UPL, 1, USK_HASH_X, GEMV>;
    case 2: return (void*)k_query_fast<E, UPL, 2, USK_HASH_X, GEMV>;
    case 3: return (void*)k_query_fast<E, UPL, 3, USK_HASH_X, GEMV>;
    default: return (void*)k_query_fast<E, UPL, 0, USK_HASH_X, GEMV>;
  }
}

template <int UPL>
void* pick_upl(bool gemv, bool bf16, int M, int hash) {
  if (gemv) return bf16 ? pick_m<uint16_t, UPL, true>(M, hash) : pick_m<uint32_t, UPL, true>(M, hash);
  return bf16 ? pick_m<uint16_t, UPL, false>(M, hash) : pick_m<uint32_t, UPL, false>(M, hash);
}

void* pick_fast(int upl, bool gemv, bool bf16, int M, int hash) {
  switch (upl) {
    case 4: return pick_upl<4>(gemv, bf16, M, hash);
    case 2: return pick_upl<2>(gemv, bf16, M, hash);
    default: return pick_upl<1>(gemv, bf16, M, hash);
  }
}

int sm_count() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) !=
                                                 cudaSuccess)
      sms = 148;
  }
  return sms;
}

int occupancy(void* kern, size_t smem) {
  // cached per (kernel, smem); the max-dynamic-smem attribute is raised on first use (callers
  // warm up before any graph capture)
  static std::mutex mu;
  static std::vector<std::pair<std::pair<void*, size_t>, int>> cache;
  static std::vector<void*> raised;
  std::lock_guard<std::mutex> lock(mu);
  for (auto& e : cache)
    if (e.first.first == kern && e.first.second == smem) return e.second;
  if (std::find(raised.begin(), raised.end(), kern) == raised.end()) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemMax) != cudaSuccess) {
      (void)cudaGetLastError();
      return 1;
    }
    raised.push_back(kern);
  }
  int occ = 1;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kQThreads, smem) != cudaSuccess || occ < 1) {
    (void)cudaGetLastError();
    occ = 1;
  }
  cache.push_back({{kern, smem}, occ});
  return occ;
}

struct Geom {
  int upl = 0;
  int maxMN = 0;
  size_t smem = 0;
  int grid = 0;
  bool one_wave = false;
  void* kern = nullptr;
  std::vector<int> n_chunks, n_sub, cpc;
};

// Units per lane: the largest UPL whose chunks all get a resident CTA (larger UPL amortises the
// per-row R broadcast and the 32-row transpose over more weights).  USK_UPL overrides (tuning).
Geom geometry(const usk_plan* pl, const int32_t* layers, const int64_t* rows, int n, bool gemv) {
  Geom G;
  for (int k = 0; k < n; ++k) G.maxMN = std::max(G.maxMN, pl->M * pl->layers[layers[k]].max_ncols);
  const int64_t in = pl->layers[layers[0]].in;
  const bool bf16 = pl->dtype == USK_BF16;
  static const int forced = [] {
    const char* e = std::getenv("USK_UPL");
    return e ? std::atoi(e) : 0;
  }();
  int best = 0, best_cap = 0;
  for (int upl : {4, 2, 1}) {
    if (forced && upl != forced) continue;
    const size_t sm = smem_bytes(upl, G.maxMN, pl->cell_bytes());
    if (sm > kSmemMax) continue;
    void* kern = pick_fast(upl, gemv, bf16, pl->M, pl->hash);
    const int cap = sm_count() * occupancy(kern, sm);
    int chunks = 0;
    for (int k = 0; k < n; ++k) chunks += (int)((in + 32 * upl - 1) / (32 * upl));
    best = upl;
    best_cap = cap;
    G.kern = kern;
    if (chunks <= cap) break;
  }
  if (!best) return G;
  G.upl = best;
  G.smem = smem_bytes(best, G.maxMN, pl->cell_bytes());
  int chunks = 0;
  for (int k = 0; k < n; ++k) {
    G.n_chunks.push_back((int)((in + 32 * best - 1) / (32 * best)));
    G.n_sub.push_back((int)((rows[k] + kSubRows - 1) / kSubRows));
    chunks += G.n_chunks.back();
  }
  // CTAs per layer ("cpc" = the layer's CTA count): one resident wave shared in proportion to
  // the layers' weights, at least one CTA per chunk and at most one per (chunk, subtile)
  double wsum = 0;
  for (int k = 0; k < n; ++k) wsum += (double)rows[k] * in;
  for (int k = 0; k < n; ++k) {
    const int share = (int)((double)best_cap * (double)rows[k] * in / std::max(wsum, 1.0));
    if (gemv) {  // cpc = CTAs per chunk (equal for every chunk; warps then balance dynamically)
      G.cpc.push_back(std::max(1, std::min(share / G.n_chunks[k], G.n_sub[k])));
      G.grid += G.cpc[k] * G.n_chunks[k];
    } else {     // cpc = CTAs of the layer, spread over its chunks
      G.cpc.push_back(std::max(G.n_chunks[k], std::min(share, G.n_chunks[k] * G.n_sub[k])));
      G.grid += G.cpc[k];
    }
  }
  G.one_wave = G.grid <= best_cap;
  return G;
}

int partial_stride(int64_t in) { return (int)((((in + 31) / 32) + 3) / 4 * 4); }

// per layer: [partials rows x CP floats][split-K counters per subtile][work counters 2 x chunks]
size_t layer_ws_counters_off(int64_t in, int64_t rows) {
  return ((size_t)rows * partial_stride(in) * 4 + 255) / 256 * 256;
}
size_t layer_ws_work_off(int64_t in, int64_t rows) {
  return layer_ws_counters_off(in, rows) + ((size_t)((rows + kSubRows - 1) / kSubRows) * 4 + 255) / 256 * 256;
}
size_t layer_ws_bytes(int64_t in, int64_t rows) {
  return layer_ws_work_off(in, rows) + ((size_t)2 * ((in + 31) / 32) * 4 + 255) / 256 * 256;
}

QArgs base_args(const usk_plan* pl, const void* sketch, int64_t in, const Geom& G) {
  QArgs A{};
  A.M = pl->M;
  A.maxMN = G.maxMN;
  A.in = in;
  A.sketch = sketch;
  A.ncols = pl->d_ncols;
  A.offsets = pl->d_offsets;
  A.ukeys = pl->d_keys;
  A.R = pl->d_R;
  A.hc = pl->hc;
  A.early_trigger = G.one_wave ? 1 : 0;
  return A;
}

usk_status launch_q(void* kern, const QArgs& A, int grid, size_t smem, bool pdl, cudaStream_t st) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(kQThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  static const bool timeline = std::getenv("USK_TIMELINE") != nullptr;  // debug / tuning only
  if (timeline) {
    static unsigned long long* dbuf = nullptr;
    if (!dbuf) USK_CUDA(cudaMalloc(&dbuf, sizeof(unsigned long long) * 4 * 8192));
    QArgs B = A;
    B.timeline = dbuf;
    USK_CUDA(cudaMemsetAsync(dbuf, 0, sizeof(unsigned long long) * 4 * grid, st));
    void* args[] = {&B};
    USK_CUDA(cudaLaunchKernelExC(&cfg, kern, args));
    std::vector<unsigned long long> h(4 * (size_t)grid);
    USK_CUDA(cudaMemcpyAsync(h.data(), dbuf, h.size() * 8, cudaMemcpyDeviceToHost, st));
    USK_CUDA(cudaStreamSynchronize(st));
    unsigned long long t0 = ~0ull, tend = 0;
    double stage = 0, comp = 0, tail = 0, last_comp = 0;
    for (int b = 0; b < grid; ++b) {
      t0 = std::min(t0, h[4 * b]);
      tend = std::max(tend, h[4 * b + 3]);
    }
    for (int b = 0; b < grid; ++b) {
      stage += (double)(h[4 * b + 1] - h[4 * b]);
      comp += (double)(h[4 * b + 2] - h[4 * b + 1]);
      tail += (double)(h[4 * b + 3] - h[4 * b + 2]);
      last_comp = std::max(last_comp, (double)(h[4 * b + 2] - t0));
    }
    double skew = 0, cmin = 1e30, cmax = 0, smax = 0;
    for (int b = 0; b < grid; ++b) {
      skew = std::max(skew, (double)(h[4 * b] - t0));
      cmin = std::min(cmin, (double)(h[4 * b + 2] - h[4 * b + 1]));
      cmax = std::max(cmax, (double)(h[4 * b + 2] - h[4 * b + 1]));
      smax = std::max(smax, (double)(h[4 * b + 1] - h[4 * b]));
    }
    std::fprintf(stderr,
                 "[usk timeline] grid=%d span=%.2fus start_skew_max=%.2fus stage mean/max=%.2f/%.2fus compute "
                 "mean/min/max=%.2f/%.2f/%.2fus tail=%.2fus last_compute_end=%.2fus\n",
                 grid, (tend - t0) / 1e3, skew / 1e3, stage / grid / 1e3, smax / 1e3, comp / grid / 1e3, cmin / 1e3,
                 cmax / 1e3, tail / grid / 1e3, last_comp / 1e3);
  } else {
    void* args[] = {const_cast<QArgs*>(&A)};
    USK_CUDA(cudaLaunchKernelExC(&cfg, kern, args));
  }
  count_launch();
  return USK_OK;
}

GenQ make_genq(const usk_plan* pl, int32_t l, const void* sketch) {
  const LayerGeom& L = pl->layers[l];
  GenQ Q{};
  Q.sketch = sketch;
  Q.ncols = pl->d_ncols;
  Q.offsets = pl->d_offsets;
  Q.ukeys = pl->d_keys;
  Q.hc = pl->hc;
  Q.unit_base = L.unit_begin;
  Q.out = L.out;
  Q.in = L.in;
  Q.M = pl->M;
  Q.gran = pl->gran;
  Q.g = pl->g;
  Q.hash = pl->hash;
  Q.es = pl->cell_bytes();
  return Q;
}

}  // namespace

size_t gemv_batch_workspace_bytes(const usk_plan* pl, const int32_t* layers, const int64_t* o0, const int64_t* o1,
                                  int n) {
  if (!fast_eligible(pl)) return 256;
  size_t b = 0;
  for (int k = 0; k < n; ++k) b += layer_ws_bytes(pl->layers[layers[k]].in, o1[k] - o0[k]);
  return std::max<size_t>(b, 256);
}

size_t gemv_workspace_bytes(const usk_plan* pl, int32_t l, int64_t o0, int64_t o1) {
  return gemv_batch_workspace_bytes(pl, &l, &o0, &o1, 1);
}

usk_status launch_gemv_batch(const usk_plan* pl, const void* sketch, const int32_t* layers, const int64_t* o0,
                             const int64_t* o1, int n, const void* x, int32_t x_dtype, void* const* y, int32_t y_dtype,
                             void* ws, cudaStream_t st) {
  std::vector<int64_t> rows(n);
  for (int k = 0; k < n; ++k) rows[k] = o1[k] - o0[k];
  Geom G = fast_eligible(pl) ? geometry(pl, layers, rows.data(), n, true) : Geom{};
  if (G.upl) {
    const int64_t in = pl->layers[layers[0]].in;
    QArgs A = base_args(pl, sketch, in, G);
    A.x = x;
    A.x_bf16 = x_dtype == USK_BF16;
    A.y_bf16 = y_dtype == USK_BF16;
    char* w = reinterpret_cast<char*>(ws);
    int cta = 0;
    for (int k = 0; k < n; ++k) {
      const size_t wsb = layer_ws_bytes(in, rows[k]);
      if (rows[k] > 0) {
        QLayer& Ly = A.layer[A.n_layers++];
        Ly.unit_base = pl->layers[layers[k]].unit_begin;
        Ly.o_begin = o0[k];
        Ly.rows = rows[k];
        Ly.n_chunks = G.n_chunks[k];
        Ly.n_sub = G.n_sub[k];
        Ly.cpc = G.cpc[k];
        Ly.cta_begin = cta;
        Ly.CP = partial_stride(in);
        cta += Ly.cpc * Ly.n_chunks;
        Ly.y = y[k];
        Ly.partial = reinterpret_cast<float*>(w);
        Ly.counters = reinterpret_cast<uint32_t*>(w + layer_ws_counters_off(in, rows[k]));
        Ly.work = reinterpret_cast<uint32_t*>(w + layer_ws_work_off(in, rows[k]));
      }
      w += wsb;
    }
    if (!A.n_layers) return USK_OK;
    return launch_q(G.kern, A, cta, G.smem, true, st);
  }
  for (int k = 0; k < n; ++k) {
    if (rows[k] == 0) continue;
    GenQ Q = make_genq(pl, layers[k], sketch);
    const int rpb = 8;
    k_gemv_gen<<<(unsigned)((rows[k] + rpb - 1) / rpb), 32 * rpb, 0, st>>>(Q, o0[k], o1[k], x, x_dtype == USK_BF16, y[k],
                                                                          y_dtype == USK_BF16);
    USK_LAUNCHED("k_gemv_gen");
  }
  return USK_OK;
}

usk_status launch_gemv(const usk_plan* pl, const void* sketch, int32_t l, const void* x, int32_t x_dtype, void* y,
                       int32_t y_dtype, int64_t o0, int64_t o1, void* ws, size_t, cudaStream_t st) {
  void* ys[1] = {y};
  return launch_gemv_batch(pl, sketch, &l, &o0, &o1, 1, x, x_dtype, ys, y_dtype, ws, st);
}

usk_status launch_reconstruct(const usk_plan* pl, const void* sketch, int32_t l, int64_t r0, int64_t r1, void* w_out,
                              int64_t ld, cudaStream_t st) {
  const LayerGeom& L = pl->layers[l];
  const int64_t rows = r1 - r0;
  if (rows == 0) return USK_OK;
  const int es = pl->cell_bytes();
  const bool aligned = ((ld * es) % 16 == 0) && (reinterpret_cast<uintptr_t>(w_out) % 16 == 0);
  Geom G = (fast_eligible(pl) && aligned) ? geometry(pl, &l, &rows, 1, false) : Geom{};
  if (G.upl) {
    QArgs A = base_args(pl, sketch, L.in, G);
    QLayer& Ly = A.layer[A.n_layers++];
    Ly.unit_base = L.unit_begin;
    Ly.o_begin = r0;
    Ly.rows = rows;
    Ly.n_chunks = G.n_chunks[0];
    Ly.n_sub = G.n_sub[0];
    Ly.cpc = G.cpc[0];
    Ly.cta_begin = 0;
    Ly.w_out = w_out;
    Ly.ld_out = ld;
    return launch_q(G.kern, A, G.grid, G.smem, false, st);
  }
  GenQ Q = make_genq(pl, l, sketch);
  const int64_t n = rows * L.in;
  k_reconstruct_gen<<<(unsigned)std::min<int64_t>((n + 255) / 256, 148 * 16), 256, 0, st>>>(Q, r0, r1, w_out, ld);
  USK_LAUNCHED("k_reconstruct_gen");
  return USK_OK;
}

usk_status launch_importance(const void* A, int32_t a_dtype, int64_t N, int64_t d, float* I, cudaStream_t st) {
  k_importance<<<(unsigned)((d + 255) / 256), 256, 0, st>>>(A, a_dtype == USK_BF16, N, d, I);
  USK_LAUNCHED("k_importance");
  return USK_OK;
}

}  // namespace usk
