// query.cu -- K3 reconstruct, K4 sketch-GEMV (decode), K6 importance.
//
// Query of one weight (Eq. 3 + Eq. 5; §3.1 "hash ... retrieved by the above
// indices in a batch ... interpreting these intermediate results"):
//   w'(o, j) = the bonded cell of maximum |.| over rows i < M (ties -> non-negative, L1/L2).
//
// Fast path (ROW granularity, one input dimension per unit), shared by K3 and K4:
//   * A launch's work items -- (layer, chunk of TJ = 32*UPL consecutive units, 16-row subtile) --
//     are laid out chunk-major; one CTA per SM computes a host-balanced contiguous item range
//     (partition_items).  A chunk's cells are one contiguous byte range: TMA bulk copies into a raw
//     shared buffer, converted shared -> shared into the bank-private rho layout
//         rho = rotl(bits_hi, 1) ^ 1 = (mag << 1) | (1 - sign)
//     with cell (i, k) of lane L's unit v at word v*32*maxMN + (i*maxN + k)*32 + L -- always bank L,
//     so the M random gathers of a warp never conflict.  The Eq. 5 select is an integer max
//     (VIMNMX3 for M=3) and rotr(rho, 1) is the IEEE pattern of -w', so the GEMV multiplies by -x
//     (exact).  The next chunk of a CTA's range is prefetched under the current one's math.
//   * Missing units of a ragged chunk point at the zero column (rho of +0) with x = 0, so the inner
//     loop has no branches.  Hash: per subtile, lanes r < 16 write the position
//     mixes R_i(o0 + r) mod 2^23 of their row to a per-warp shared table (one 16-B broadcast load
//     per row); per weight and sketch row one LOP3 (R_i ^ key), one FFMA.RZ (short-unit index +
//     slot offset, exact) and one IMAD (x128 + lane base) give the bank-private shared address.
//   * K4 (k_gemv_fast + k_gemv_reduce): per subtile a transpose butterfly leaves one row sum per
//     lane; chunk partials go to a row-major [rows][CP] workspace and a second, PDL-chained kernel
//     sums them in fixed order (deterministic, no float atomics).  The sketch is staged before
//     griddepcontrol.wait; x is read after it.  usk_linear_batch puts several linears that share x
//     (q|k|v, gate|up) in one call.
//   * K3 (k_recon_fast): the same skeleton storing W' rows (8-byte stores for bf16, UPL = 4).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <tuple>

#include "common.cuh"
#include "ptx.cuh"

namespace usk {
namespace {

#ifndef USK_QUERY_LOPADDR
#define USK_QUERY_LOPADDR 1
#endif
#ifndef USK_QUERY_THREADS
#define USK_QUERY_THREADS 512
#endif
constexpr int kQThreads = USK_QUERY_THREADS;
constexpr int kMaxBatch = 8;
constexpr int kMaxCtas = 256;  // GEMV compute grid (one CTA per SM)
// USK_TRACE stamps per CTA: start, staged (first segment: + wait + x), compute done, exit; first bulk
// copy issued, first piece landed, first segment converted, griddepcontrol.wait returned
constexpr int kTS = 8;
#ifndef USK_SUB_ROWS
#define USK_SUB_ROWS 16
#endif
constexpr int kSubRows = USK_SUB_ROWS;  // rows per warp work item (subtile) of the default kernels: 8 or 16
static_assert(kSubRows == 8 || kSubRows == 16, "subtile rows");
// The raw-bf16 GEMV is also built with 8-row subtiles: the host picks them for calls whose 16-row
// items would leave the last round of a CTA's warps mostly idle (q|k|v, down of Llama-3.2-1B).
constexpr int kRTabWordOffset = 32 + 160;  // zero cells + chunk unit offsets (<= 129)
constexpr int kRTabWords = (kQThreads / 32) * 16 * 4;  // per warp: up to 16 rows x {R_0, R_1, R_2, 0}
constexpr int kCellsWordOffset = kRTabWordOffset + kRTabWords;

extern __shared__ __align__(16) uint32_t qsm[];  // dynamic shared memory of the query kernels

// 32-bit shared load at a shared-window byte address (ld.shared: no generic -> shared conversion
// in the inner loop).
__device__ __forceinline__ uint32_t lds_at(uint32_t saddr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(saddr));
  return v;
}

struct QLayer {
  int64_t unit_base;   // global unit id of the layer's first unit
  int64_t o_begin;     // first output row
  int64_t rows;        // rows in [o_begin, o_end)
  int64_t item_begin;  // GEMV: first work item (chunk-major, subtile-minor) of the layer in the launch
  int64_t row_begin;   // GEMV: first row of the layer in the launch's reduction order
  int32_t n_chunks;    // unit chunks of TJ
  int32_t n_sub;       // 16-row subtiles
  int32_t CP;          // GEMV: row stride of the partial workspace (>= n_chunks, multiple of 4)
  int32_t pad;
  void* y;             // GEMV output
  float* partial;      // GEMV: [rows][CP] chunk partials
  void* w_out;         // reconstruct output
  int64_t ld_out;
  const int32_t* oidx; // Top-K side table: ascending flat indices o*in + j (global rows), or NULL
  const void* ovals;   //   their states (plan dtype)
  int64_t n_out;
  int64_t out_rows;    // out_features of the layer (flat index stride is `in`)
};

struct QArgs {
  QLayer layer[kMaxBatch];
  int32_t n_layers;
  int32_t M;
  int32_t maxMN;        // smem slot stride (cells) = M * maxN
  int32_t piece_units;  // units per bulk copy when staging a chunk (power of two, <= TJ)
  int32_t maxN;         // smem stride (cells) between sketch rows of a slot: 1 + max N over the
                        // launch's units; column maxN - 1 of every row holds rho(+0) (zero column)
  uint32_t row_bytes;   // 128 * maxN: shared byte distance between sketch rows of a slot
  int64_t in;           // in_features (shared by the batch)
  int64_t items;        // GEMV: total work items (chunk, subtile) of the launch
  int64_t rows;         // GEMV: total output rows of the launch
  const void* sketch;
  const int32_t* ncols;
  const uint8_t* nrows;  // M_u per unit (<= M; ledger L30): staged rows >= M_u hold rho = 0 (neutral)
  const int64_t* offsets;
  const uint32_t* ukeys;
  HashConsts hc;
  const void* x;
  int32_t x_bf16;
  int32_t y_bf16;
  int32_t red_lanes;               // GEMV reduce: lanes per row (power of two <= 32)
  int32_t g_shift;                 // quantised plans: log2(group size)
  int32_t sbuf_off;                // quantised plans: byte offset of the staged scales from the raw buffer
  const float* scales;             // quantised plans: fp32 group scales (in the sketch buffer)
  int32_t es;                      // bytes of a raw state (Top-K side-table values)
  int32_t cta_item[kMaxCtas + 1];  // GEMV: CTA c computes work items [cta_item[c], cta_item[c + 1])
  // raw plans: CTA c's first bulk copy, precomputed on the host from the plan's unit offsets (no
  // dependent global load before it): 16-B aligned sketch byte offset | copy shift (low 4 bits), bytes
  int32_t first_ok;
  uint64_t first_a0s[kMaxCtas];
  uint32_t first_bytes[kMaxCtas];
  unsigned long long* timeline;  // tuning only (USK_TRACE): kTS globaltimer stamps per CTA
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

template <int MT, int HASH>
constexpr bool fast_hash() { return MT > 0 && HASH == USK_HASH_X; }

// Raw bf16 plans stage "key|value" cell words: the high half is the 16-bit retrieve key
// rho16 = rotl16(b, 1) ^ 1 = (mag << 1) | (1 - sign), the low half the state's bf16 bits b.  An
// unsigned max over words is decided by the keys (equal keys = equal bits), so the Eq. 5 select
// is one VIMNMX3 and the selected word's low half IS w' in bf16: the GEMV multiplies it directly
// (fma.rn.f32.bf16, exact product and one rounding, the same bits as an fp32 FFMA of the
// widened operands) and the reconstruction stores it as it is.  fp32 and quantised plans keep
// 32-bit rho words (rotl(bits, 1) ^ 1; rotr(rho, 1) = bits of -w').
template <typename E, int QB>
constexpr bool kv_cells() { return sizeof(E) == 2 && QB == 0; }

__device__ __forceinline__ uint32_t kv_word(uint32_t b16) {
  return ((((b16 << 1) | (b16 >> 15)) & 0xFFFFu) ^ 1u) << 16 | b16;
}

// c + bf16(xb) * bf16(low half of w): one FHFMA.BF16
__device__ __forceinline__ float fma_bf16_lo(uint32_t xb, uint32_t w, float c) {
  float d;
  asm("{.reg .b16 wl, wh, xl, xh;\n\t"
      "mov.b32 {wl, wh}, %2;\n\t"
      "mov.b32 {xl, xh}, %1;\n\t"
      "fma.rn.f32.bf16 %0, xl, wl, %3;}"
      : "=f"(d)
      : "r"(xb), "r"(w), "f"(c));
  return d;
}

template <int UPL, int MT, int HASH>
struct LaneState {
  static constexpr int KR = fast_hash<MT, HASH>() ? MT : 1;
  // generic (M > 3, identity hash): unit key, N and the shared-window byte address of (unit v,
  // sketch row 0, column 0) for this lane; cell (i, k) is at b0 + 128 * (i * maxN + k)
  uint32_t K[UPL], N[UPL], b0[UPL];
  // fast: FFMA key and addend of (unit v, sketch row i); address = bits * 128 + B
  uint32_t fk[UPL][KR], cb[UPL][KR];
  float Nf[UPL];
  uint32_t B;
#if USK_QUERY_LOPADDR
  // M = 3: sketch row 2 takes its address from an ALU-pipe LOP3 instead of an FMA-pipe IMAD (the two
  // pipes then carry 6 + 6 of the 15 instructions per 32 weights): FFMA.RZ(f, 128 N, 2^23 + B2 - 128 N)
  // rounds to 2^23 + B2 + floor(128 k N / 2^23) (ulp 1), and masking its mantissa to bits 7..22 leaves
  // B2 + 128 idx; cb[v][2] holds those addend bits, B2 = the 128-aligned byte address of the slot row
  float Nf128[UPL];
  uint32_t L4;  // 4 * lane (the cells start 128-B aligned)
#endif
};

// the rho cells start at a 128-B aligned shared address (row 2's LOP3 address keeps the lane bits)
__device__ __forceinline__ uint32_t* q_cells() {
  const uint32_t a = smem_u32(qsm + kCellsWordOffset);
  return qsm + kCellsWordOffset + ((128u - (a & 127u)) & 127u) / 4u;
}

// shared memory: [zero cells: 32 words][mbarrier: 2 words][copy shift: 1 word]...[per-warp R tables
// @ word kRTabWordOffset][cells @ word kCellsWordOffset: UPL*32*maxMN words][raw bulk-copy buffer:
// piece_units*maxMN cells + 32 B]
__device__ __forceinline__ uint64_t* q_bar() { return reinterpret_cast<uint64_t*>(qsm + 32); }

// Lane state of a chunk [ubase, ubase + nu): keys, N_u and the shared addresses of each of the
// lane's units (missing units of a ragged chunk point at the zero cells: idx is always 0).
template <int UPL, int MT, int HASH>
__device__ __forceinline__ void lane_setup(const QArgs& A, int64_t ubase, int nu, LaneState<UPL, MT, HASH>& S) {
  const int lane = threadIdx.x & 31;
  const uint32_t cbase = smem_u32(q_cells());
  S.B = cbase + 4u * (uint32_t)lane;  // (0x4C000000 << 7) wraps to 0
#if USK_QUERY_LOPADDR
  S.L4 = 4u * (uint32_t)lane;
#endif
#pragma unroll
  for (int v = 0; v < UPL; ++v) {
    const int ul = UPL * lane + v;
    const bool valid = ul < nu;
    if (valid) {
      S.K[v] = A.ukeys[ubase + ul];
      S.N[v] = (uint32_t)A.ncols[ubase + ul];
      S.b0[v] = cbase + 4u * (uint32_t)(v * 32 * A.maxMN + lane);
    } else {  // missing unit of a ragged chunk: idx is always 0 -> the zero column of every row
      S.K[v] = 0;
      S.N[v] = 1;
      S.b0[v] = cbase + 4u * (uint32_t)((A.maxN - 1) * 32 + lane);
    }
    S.Nf[v] = (float)(4u * S.N[v]);
    if constexpr (fast_hash<MT, HASH>()) {
#pragma unroll
      for (int i = 0; i < MT; ++i) {
        S.fk[v][i] = short_fkey(row_key(S.K[v], A.hc.kap[i]));
        S.cb[v][i] = short_cbits(S.N[v], valid ? (uint32_t)(v * A.maxMN + i * A.maxN) : (uint32_t)(i * A.maxN + A.maxN - 1));
      }
#if USK_QUERY_LOPADDR
      if constexpr (MT == 3) {
        const uint32_t off2 = valid ? (uint32_t)(v * A.maxMN + 2 * A.maxN) : (uint32_t)(3 * A.maxN - 1);
        S.Nf128[v] = (float)(128u * S.N[v]);
        S.cb[v][2] = __float_as_uint((float)(8388608u + cbase + 128u * off2 - 128u * S.N[v]));  // exact (< 2^24)
      }
#endif
    }
  }
}

template <typename E, int UPL>
__device__ __forceinline__ unsigned char* q_raw(const QArgs& A) {
  return reinterpret_cast<unsigned char*>(q_cells() + UPL * 32 * A.maxMN);
}

// thread 0: bulk copy of the cells of units [ubase + pa, ubase + pa + pn) into the raw buffer.
// Quantised plans (QB = 4 / 8 bits, L25): the cells' packed codes into the raw buffer and
// their groups' fp32 scales into the scale buffer, both on the same mbarrier.
template <typename E, int UPL, int QB>
__device__ __forceinline__ void stage_issue(const QArgs& A, int64_t ubase, int pa, int pn) {
  constexpr int ES = sizeof(E);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // earlier generic reads of raw
  if constexpr (QB == 0) {
    const uint64_t g0 = (uint64_t)A.offsets[ubase + pa] * ES, g1 = (uint64_t)A.offsets[ubase + pa + pn] * ES;
    const uint64_t a0 = g0 & ~uint64_t(15), a1 = (g1 + 15) & ~uint64_t(15);
    mbar_arrive_expect_tx(q_bar(), (uint32_t)(a1 - a0));
    bulk_g2s(q_raw<E, UPL>(A), reinterpret_cast<const unsigned char*>(A.sketch) + a0, (uint32_t)(a1 - a0), q_bar());
    qsm[34] = (uint32_t)(g0 - a0);  // copy shift
  } else {
    const int64_t c0 = A.offsets[ubase + pa], c1 = A.offsets[ubase + pa + pn];
    const uint64_t a0 = ((uint64_t)c0 * QB / 8) & ~uint64_t(15), a1 = (((uint64_t)c1 * QB + 7) / 8 + 15) & ~uint64_t(15);
    const uint64_t s0 = ((uint64_t)(c0 >> A.g_shift) * 4) & ~uint64_t(15);
    const uint64_t s1 = ((uint64_t)(((c1 - 1) >> A.g_shift) + 1) * 4 + 15) & ~uint64_t(15);
    mbar_arrive_expect_tx(q_bar(), (uint32_t)((a1 - a0) + (s1 - s0)));
    bulk_g2s(q_raw<E, UPL>(A), reinterpret_cast<const unsigned char*>(A.sketch) + a0, (uint32_t)(a1 - a0), q_bar());
    bulk_g2s(q_raw<E, UPL>(A) + A.sbuf_off, reinterpret_cast<const unsigned char*>(A.scales) + s0, (uint32_t)(s1 - s0),
             q_bar());
    reinterpret_cast<uint64_t*>(qsm + 34)[0] = a0;      // byte of code storage at raw[0]
    reinterpret_cast<uint64_t*>(qsm + 36)[0] = s0 / 4;  // group of scale buffer entry 0
  }
}

// Stage the cells of units [ubase, ubase + nu) (consecutive in the sketch, so contiguous bytes)
// into the bank-private rho layout: pieces of piece_units units are brought in by one TMA bulk
// copy each (cp.async.bulk, mbarrier completion) and converted shared -> shared.  The first
// piece may have been issued already (first_issued; thread 0 called stage_issue).  Ends with a
// __syncthreads (cells complete, raw buffer free).  The mbarrier phase advances once per piece.
// Quantised plans convert each cell to its dequantised value fl32(code * scale) first, so the
// query loop is the same for every plan (the rho of an fp32 value).
template <typename E, int UPL, int QB>
__device__ __forceinline__ void stage_units(const QArgs& A, int64_t ubase, int nu, uint32_t& phase,
                                            bool first_issued, unsigned long long* landed = nullptr) {
  constexpr int ES = sizeof(E);
  uint32_t* cells = q_cells();
  const unsigned char* raw = q_raw<E, UPL>(A);
  const int pu = A.piece_units;
  for (int pa = 0; pa < nu; pa += pu) {
    const int pn = min(pu, nu - pa);
    if (threadIdx.x == 0 && !(pa == 0 && first_issued)) stage_issue<E, UPL, QB>(A, ubase, pa, pn);
    // thread -> unit of the piece: for pu >= 32 a warp's 32 lanes take units pu/32 apart, so their
    // cells land in distinct owner lanes ul / UPL (banks) -- conflict-free stores for pu = 32 * UPL
    const int tt = threadIdx.x & (pu - 1);
    const int t = pu >= 32 ? (tt & 31) * (pu >> 5) + (tt >> 5) : tt;
    const int ul = pa + t;
    int64_t u_off = 0, cu = 0;
    int n = 0;  // N of the thread's unit (0: no unit)
    int m = 0;  // M_u of the thread's unit: slot rows >= m get rho = 0, the identity of the max
    if (t < pn) {  // overlaps the copy
      cu = A.offsets[ubase + ul];
      u_off = cu - A.offsets[ubase + pa];
      n = A.ncols[ubase + ul];
      m = A.nrows[ubase + ul];
    }
    __syncthreads();  // shift visible
    mbar_wait(q_bar(), phase);
    phase ^= 1u;
    if (landed && pa == 0 && threadIdx.x == 0) *landed = gtimer();
    uint32_t* dst = cells + (ul % UPL) * 32 * A.maxMN + ul / UPL;
    const int KS = kQThreads / pu;
    if constexpr (QB == 0) {
      const unsigned char* src = raw + qsm[34] + u_off * ES;
      for (int i = 0; i < A.M; ++i, src += n * ES, dst += A.maxN * 32) {  // sketch row i -> slot row i
        if (i >= m) {
          for (int k = threadIdx.x / pu; k < n; k += KS) dst[k * 32] = 0u;
          continue;
        }
#pragma unroll 2
        for (int k = threadIdx.x / pu; k < n; k += KS) {
          if constexpr (ES == 2) {
            dst[k * 32] = kv_word(reinterpret_cast<const uint16_t*>(src)[k]);
          } else {
            dst[k * 32] = rotl1(reinterpret_cast<const uint32_t*>(src)[k]) ^ 1u;
          }
        }
      }
    } else {
      const uint64_t a0 = reinterpret_cast<const uint64_t*>(qsm + 34)[0];
      const uint64_t sg0 = reinterpret_cast<const uint64_t*>(qsm + 36)[0];
      const float* sb = reinterpret_cast<const float*>(raw + A.sbuf_off);
      for (int i = 0; i < A.M; ++i, dst += A.maxN * 32) {
        if (i >= m) {
          for (int k = threadIdx.x / pu; k < n; k += KS) dst[k * 32] = 0u;
          continue;
        }
#pragma unroll 4
        for (int k = threadIdx.x / pu; k < n; k += KS) {
          const int64_t c = cu + (int64_t)i * n + k;  // global cell
          int code;
          if constexpr (QB == 8) {
            code = (int)(int8_t)raw[(uint64_t)c - a0];
          } else {
            const uint32_t byte = raw[((uint64_t)c >> 1) - a0];
            code = (int)((byte >> ((c & 1) * 4)) & 0xFu);
            code = (code ^ 8) - 8;  // sign-extend the nibble
          }
          const float v = __fmul_rn((float)code, sb[((uint64_t)c >> A.g_shift) - sg0]);
          dst[k * 32] = rotl1(__float_as_uint(v)) ^ 1u;
        }
      }
    }
    __syncthreads();
  }
}

// kernel prologue shared by the fast kernels: zero column of every slot row, staging mbarrier
template <int UPL, bool KV>
__device__ __forceinline__ void q_prologue(const QArgs& A, bool init_bar = true) {
  uint32_t* cells = q_cells();
  for (int e = threadIdx.x; e < UPL * A.M * 32; e += kQThreads) {
    const int lane = e & 31, vi = e >> 5, v = vi % UPL, i = vi / UPL;
    cells[v * 32 * A.maxMN + (i * A.maxN + A.maxN - 1) * 32 + lane] = KV ? 0x00010000u : 1u;  // +0
  }
  if (threadIdx.x == 0 && init_bar) {
    mbar_init(q_bar(), 1);
    fence_mbar_init();
  }
}

// rho code of w'(o, unit v) for this lane; R = the row's position mixes R_i(o) mod 2^23 (fast hash)
template <int UPL, int MT, int HASH>
__device__ __forceinline__ uint32_t select_rho(const QArgs& A, const LaneState<UPL, MT, HASH>& S, int v, const uint4& R,
                                               int64_t o) {
  if constexpr (fast_hash<MT, HASH>()) {
    const uint32_t Ri[3] = {R.x, R.y, R.z};
    uint32_t m[MT];
#if USK_QUERY_LOPADDR
    if constexpr (MT == 3) {
      m[0] = lds_at(short_fma_bits(Ri[0], S.fk[v][0], S.Nf[v], S.cb[v][0]) * 128u + S.B);
      m[1] = lds_at(short_fma_bits(Ri[1], S.fk[v][1], S.Nf[v], S.cb[v][1]) * 128u + S.B);
      uint32_t a2;  // (bits & 0x7FFF80) | lane bits: one LOP3
      asm("lop3.b32 %0, %1, 0x7FFF80, %2, 0xEA;" : "=r"(a2) : "r"(short_fma_bits(Ri[2], S.fk[v][2], S.Nf128[v], S.cb[v][2])), "r"(S.L4));
      m[2] = lds_at(a2);
    } else
#endif
    {
#pragma unroll
      for (int i = 0; i < MT; ++i) m[i] = lds_at(short_fma_bits(Ri[i], S.fk[v][i], S.Nf[v], S.cb[v][i]) * 128u + S.B);
    }
    uint32_t best = m[0];
#pragma unroll
    for (int i = 1; i < MT; ++i) best = max(best, m[i]);
    return best;
  } else {
    uint32_t best = 0;
    for (int i = 0; i < A.M; ++i) {
      const uint32_t idx = (HASH == USK_HASH_X) ? hash_index_x(A.hc, (uint32_t)o, S.K[v], i, S.N[v])
                                                : (uint32_t)(o % S.N[v]);
      best = max(best, lds_at(S.b0[v] + ((idx + i * A.maxN) << 7)));
    }
    return best;
  }
}

// per-warp table of the subtile rows' position mixes: lane r < kSubRows writes row r's
// {R_0, R_1, R_2} mod 2^23 (rows past the layer repeat its last row)
template <int MT, int HASH, int SR>
__device__ __forceinline__ void fill_rtab(const QArgs& A, uint32_t rtab, int64_t o_first, int64_t o_last, int lane) {
  if constexpr (fast_hash<MT, HASH>()) {
    __syncwarp();  // the previous subtile's reads are done
    if (lane < SR) {
      const uint32_t o = (uint32_t)min(o_first + lane, o_last);
      const uint32_t r0 = fmix32(o ^ A.hc.rho[0]) & 0x7FFFFFu;
      const uint32_t r1 = MT > 1 ? fmix32(o ^ A.hc.rho[1]) & 0x7FFFFFu : 0u;
      const uint32_t r2 = MT > 2 ? fmix32(o ^ A.hc.rho[2]) & 0x7FFFFFu : 0u;
      asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(rtab + 16u * lane), "r"(r0), "r"(r1), "r"(r2),
                   "r"(0u) : "memory");
    }
    __syncwarp();
  }
}

__device__ __forceinline__ uint4 lds_rtab(uint32_t a) {
  uint4 q;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(q.x), "=r"(q.y), "=r"(q.z), "=r"(q.w) : "r"(a));
  return q;
}

// Row sums of a subtile: acc[r] is this lane's partial of row r.  Every row is summed over the 32
// lanes by ONE fixed tree whatever the subtile height: lane bits 3, 2, 1, 0, then 4, each stage
// adding the partial of the lane across that bit (fp addition commutes, so the two lanes of a pair
// agree).  16-row subtiles: exchange-and-halve stages on lane bits 3..0 (row bit 3..0), then bit 4;
// 8-row subtiles: exchange stages on lane bits 3, 2, 1 (row bits 2, 1, 0), then bits 0 and 4.  So a
// row's bits do not depend on the subtile height (a per-launch choice), its position in the
// subtile, the output range, the batch or the GPU count (bit-identical shards).
// Returns the sum of row sub_row<SR>(lane) (replicated over the lanes that share it).
template <int SR>
__device__ __forceinline__ int sub_row(int lane) { return SR == 16 ? (lane & 15) : ((lane >> 1) & 7); }
template <int SR>
__device__ __forceinline__ bool row_writer(int lane) { return SR == 16 ? lane < 16 : (lane & 17) == 0; }

template <int SR>
__device__ __forceinline__ float transpose_reduce(float (&acc)[SR], int lane) {
  static_assert(SR == 8 || SR == 16, "subtile rows");
  constexpr int LS = SR == 16 ? 1 : 2;  // lane distance of row bit b: LS << b
#pragma unroll
  for (int m = SR / 2; m >= 1; m >>= 1) {
    const bool up = (lane & (LS * m)) != 0;
#pragma unroll
    for (int i = 0; i < m; ++i) {
      const float send = up ? acc[i] : acc[i + m];
      const float keep = up ? acc[i + m] : acc[i];
      acc[i] = keep + __shfl_xor_sync(0xffffffffu, send, LS * m);
    }
  }
  float t = acc[0];
  if constexpr (SR == 8) t += __shfl_xor_sync(0xffffffffu, t, 1);
  t += __shfl_xor_sync(0xffffffffu, t, 16);
  return t;
}

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

#ifndef USK_QUERY_MINB
#define USK_QUERY_MINB 1
#endif
#ifndef USK_GEMV_MAXREG
#define USK_GEMV_MAXREG 112  // 512 x 112 + 256 x 32 registers: k_gemv_fast + k_gemv_reduce share an SM
#endif

// store the UPL reconstructed weights (fp32 bit patterns; raw bf16 plans: bf16 bits in the high
// half, exact) of lane L's units.  RNE: quantised plans round the fp32 dequantised value to bf16
// (round to nearest even, L25); raw bf16 plans take the high half as it is.
template <typename E, int UPL, bool RNE, bool LO = false>
__device__ __forceinline__ void store_units(E* dst, uint32_t (&wb)[UPL], bool full_tile, int nu, int lane) {
  if constexpr (LO) {  // key|value words: the bf16 bits are the low halves
    if (full_tile) {
      if constexpr (UPL == 4) {
        *reinterpret_cast<uint2*>(dst) = make_uint2(__byte_perm(wb[0], wb[1 % UPL], 0x5410),
                                                    __byte_perm(wb[2 % UPL], wb[3 % UPL], 0x5410));
      } else if constexpr (UPL == 2) {
        *reinterpret_cast<uint32_t*>(dst) = __byte_perm(wb[0], wb[1 % UPL], 0x5410);
      } else {
        dst[0] = (E)(wb[0] & 0xFFFFu);
      }
    } else {
#pragma unroll
      for (int v = 0; v < UPL; ++v)
        if (UPL * lane + v < nu) dst[v] = (E)(wb[v] & 0xFFFFu);
    }
    return;
  }
  if constexpr (sizeof(E) == 2 && RNE) {
#pragma unroll
    for (int v = 0; v < UPL; ++v) wb[v] = wb[v] + 0x7FFFu + ((wb[v] >> 16) & 1u);
  }
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

// ------------------------------------------------------------------ K4: sketch-GEMV (decode)
// Two kernels per call, chained with programmatic dependent launch (no grid barrier):
//  * k_gemv_fast (one CTA per SM): the launch's work items (layer, chunk, subtile) are laid out
//    chunk-major and CTA c computes the contiguous range [cta_item[c], cta_item[c+1]) -- the host
//    balances the ranges, charging every chunk boundary inside a range for its extra staging.
//    Warps grab the subtiles of a staged chunk dynamically; the next chunk of the range is
//    prefetched (TMA) under the current one's math.  Chunk partials go to [rows][CP].
//  * k_gemv_reduce: y[r] = the fixed-order sum of row r's chunk partials.  Its small CTAs fit
//    beside k_gemv_fast's (register budget 112 + 32 per thread), wait there for the partials
//    (griddepcontrol.wait), and the NEXT call's k_gemv_fast stages its sketch chunk while they
//    reduce.
template <typename E, int UPL, int MT, int HASH, bool GEMV, int QB, bool XB, int SR = kSubRows>
__device__ __forceinline__ void query_balanced(const QArgs& A) {
  constexpr int TJ = 32 * UPL;
  constexpr bool KV = kv_cells<E, QB>();
  __shared__ int s_next;  // next subtile of the current segment (warps grab dynamically)
  const int lane = threadIdx.x & 31;
  const int c = blockIdx.x;
  const int64_t s_begin = A.cta_item[c], s_end = A.cta_item[c + 1];
  if (A.timeline && threadIdx.x == 0) A.timeline[c * kTS + 0] = gtimer();
  const bool pre = QB == 0 && A.first_ok && s_begin < s_end;
  if (pre && threadIdx.x == 0) {  // first piece in flight before anything else
    const uint64_t a0s = A.first_a0s[c];
    const uint32_t bytes = A.first_bytes[c];
    mbar_init(q_bar(), 1);
    fence_mbar_init();
    mbar_arrive_expect_tx(q_bar(), bytes);
    bulk_g2s(q_raw<E, UPL>(A), reinterpret_cast<const unsigned char*>(A.sketch) + (a0s & ~uint64_t(15)), bytes, q_bar());
    qsm[34] = (uint32_t)(a0s & 15u);  // copy shift
  }
  q_prologue<UPL, KV>(A, !pre);
  uint32_t phase = 0;
  bool waited = false;
  // a segment = the part of [s_begin, s_end) inside one chunk
  struct Seg {
    int li, chunk, sub_a, sub_end, nu;
    int64_t end, j0, ubase;
  };
  auto seg_at = [&](int64_t s) {
    Seg g;
    g.li = 0;
    while (g.li + 1 < A.n_layers && A.layer[g.li + 1].item_begin <= s) ++g.li;
    const QLayer& L = A.layer[g.li];
    const int64_t local = s - L.item_begin;
    g.chunk = (int)(local / L.n_sub);
    g.sub_a = (int)(local - (int64_t)g.chunk * L.n_sub);
    g.end = min(s_end, L.item_begin + (int64_t)(g.chunk + 1) * L.n_sub);
    g.sub_end = g.sub_a + (int)(g.end - s);
    g.j0 = (int64_t)g.chunk * TJ;
    g.nu = (int)min((int64_t)TJ, A.in - g.j0);
    g.ubase = L.unit_base + g.j0;
    return g;
  };
  if (s_begin < s_end) {
    Seg cur = seg_at(s_begin);
    if (threadIdx.x == 0) {
      s_next = cur.sub_a;
      if (!pre) stage_issue<E, UPL, QB>(A, cur.ubase, 0, min(A.piece_units, cur.nu));  // first piece in flight
      if (A.timeline) A.timeline[c * kTS + 4] = gtimer();
    }
    bool stamped = false;
    while (true) {
      const QLayer& Ly = A.layer[cur.li];
      LaneState<UPL, MT, HASH> S;
      lane_setup<UPL, MT, HASH>(A, cur.ubase, cur.nu, S);  // overlaps the copy
      stage_units<E, UPL, QB>(A, cur.ubase, cur.nu, phase, true,
                              (A.timeline && !waited) ? A.timeline + c * kTS + 5 : nullptr);  // sketch only: before the wait
      if (!waited) {
        if (A.timeline && threadIdx.x == 0) A.timeline[c * kTS + 6] = gtimer();
        pdl_wait();     // x may be written by the previous kernel on the stream
        pdl_trigger();  // every CTA of this grid is running: the next launch may be scheduled
        if (A.timeline && threadIdx.x == 0) A.timeline[c * kTS + 7] = gtimer();
        waited = true;
      }
      float nx[UPL];    // rho words: -x (rotr(rho) decodes to -w'); key|value words: x
      uint32_t xb[UPL];  // XB: x as bf16 bits (fma.rn.f32.bf16 operand)
#pragma unroll
      for (int v = 0; v < UPL; ++v) {
        const int64_t j = cur.j0 + UPL * lane + v;
        float xv = 0.f;
        xb[v] = 0u;
        if (GEMV && UPL * lane + v < cur.nu) {
          if constexpr (XB) {
            xb[v] = reinterpret_cast<const uint16_t*>(A.x)[j];
          } else {
            xv = A.x_bf16 ? __uint_as_float((uint32_t)reinterpret_cast<const uint16_t*>(A.x)[j] << 16)
                          : reinterpret_cast<const float*>(A.x)[j];
          }
        }
        nx[v] = KV ? xv : -xv;
      }
      if (A.timeline && threadIdx.x == 0 && !stamped) A.timeline[c * kTS + 1] = gtimer();
      stamped = true;
      // the raw buffer is free: prefetch the next segment's first piece under this one's math
      const bool more = cur.end < s_end;
      Seg nxt_seg = cur;
      if (more) {
        nxt_seg = seg_at(cur.end);
        if (threadIdx.x == 0) stage_issue<E, UPL, QB>(A, nxt_seg.ubase, 0, min(A.piece_units, nxt_seg.nu));
      }
      auto next_sub = [&]() -> int {
        int g = 0;
        if (lane == 0) g = atomicAdd(&s_next, 1);
        return __shfl_sync(0xffffffffu, g, 0);
      };
      const int sub_end = cur.sub_end;
      const int chunk = cur.chunk;
      const uint32_t rtab = smem_u32(qsm + kRTabWordOffset) + (uint32_t)(threadIdx.x >> 5) * (16u * 16u);
      int sub = next_sub();
      if (sub < sub_end) fill_rtab<MT, HASH, SR>(A, rtab, Ly.o_begin + (int64_t)sub * SR, Ly.o_begin + Ly.rows - 1, lane);
      while (sub < sub_end) {
        const int nxt = next_sub();  // issued now, consumed after this subtile's math
        const int64_t r0 = (int64_t)sub * SR;
        const int nrow = (int)min((int64_t)SR, Ly.rows - r0);
        if constexpr (GEMV) {
          float acc[SR];
#pragma unroll
          for (int r = 0; r < SR; ++r) {
            uint4 Rv = make_uint4(0, 0, 0, 0);
            if constexpr (fast_hash<MT, HASH>()) Rv = lds_rtab(rtab + 16u * r);
            float a = 0.f;
#pragma unroll
            for (int v = 0; v < UPL; ++v) {
              const uint32_t wsel = select_rho<UPL, MT, HASH>(A, S, v, Rv, Ly.o_begin + r0 + r);
              if constexpr (KV && XB) a = fma_bf16_lo(xb[v], wsel, a);
              else if constexpr (KV) a = fmaf(nx[v], __uint_as_float(wsel << 16), a);
              else a = fmaf(nx[v], __uint_as_float(rotr1(wsel)), a);
            }
            acc[r] = a;
          }
          const float t = transpose_reduce<SR>(acc, lane);
          if constexpr (SR == 16) {
            if (lane < nrow) Ly.partial[(r0 + lane) * Ly.CP + chunk] = t;
          } else {
            const int rr = sub_row<SR>(lane);
            if (row_writer<SR>(lane) && rr < nrow) Ly.partial[(r0 + rr) * Ly.CP + chunk] = t;
          }
        } else {
          // W' rows: lane L writes its UPL units of each row (bf16: one 8-byte store for UPL = 4)
          const bool full_tile = (cur.nu == TJ);
          E* dst = reinterpret_cast<E*>(Ly.w_out) + r0 * Ly.ld_out + cur.j0 + UPL * lane;
#pragma unroll 4
          for (int r = 0; r < SR; ++r, dst += Ly.ld_out) {
            if (r >= nrow) continue;
            uint4 Rv = make_uint4(0, 0, 0, 0);
            if constexpr (fast_hash<MT, HASH>()) Rv = lds_rtab(rtab + 16u * r);
            uint32_t wb[UPL];
#pragma unroll
            for (int v = 0; v < UPL; ++v) {
              const uint32_t wsel = select_rho<UPL, MT, HASH>(A, S, v, Rv, Ly.o_begin + r0 + r);
              wb[v] = KV ? wsel : rotr1(wsel) ^ 0x80000000u;  // key|value: bf16 in the low half
            }
            store_units<E, UPL, QB != 0, KV>(dst, wb, full_tile, cur.nu, lane);
          }
        }
        sub = nxt;
        if (sub < sub_end) fill_rtab<MT, HASH, SR>(A, rtab, Ly.o_begin + (int64_t)sub * SR, Ly.o_begin + Ly.rows - 1, lane);
      }
      __syncthreads();  // cells and s_next are reused by the next segment
      if (!more) break;
      cur = nxt_seg;
      if (threadIdx.x == 0) s_next = cur.sub_a;
    }
  }
  if (!waited) {
    pdl_wait();
    pdl_trigger();
  }
  if (A.timeline && lane == 0) {
    atomicMax(&A.timeline[c * kTS + 2], gtimer());
    atomicMax(&A.timeline[c * kTS + 3], gtimer());
  }
}

template <typename E, int UPL, int MT, int HASH, int QB, bool XB, int SR = kSubRows>
__global__ void __maxnreg__(USK_GEMV_MAXREG) k_gemv_fast(const __grid_constant__ QArgs A) {
  query_balanced<E, UPL, MT, HASH, true, QB, XB, SR>(A);
}

// K3 fast path: the same balanced chunk-major partition, staging and per-subtile select as
// k_gemv_fast, with W' rows stored instead of multiplied (no x, no reduction).
template <typename E, int UPL, int MT, int HASH, int QB>
__global__ void __maxnreg__(USK_GEMV_MAXREG) k_recon_fast(const __grid_constant__ QArgs A) {
  query_balanced<E, UPL, MT, HASH, false, QB, false>(A);
}

// Top-K (L29): [lo, hi) of the side-table entries of global row o
__device__ __forceinline__ void outlier_range(const int32_t* idx, int64_t n, int64_t o, int64_t in, int64_t& lo,
                                              int64_t& hi) {
  auto lower = [&](int64_t key) {
    int64_t a = 0, b = n;
    while (a < b) {
      const int64_t m = (a + b) >> 1;
      if ((int64_t)(uint32_t)idx[m] < key) a = m + 1;
      else b = m;
    }
    return a;
  };
  lo = lower(o * in);
  hi = lower((o + 1) * in);
}

__device__ __forceinline__ float state_value(const void* vals, int32_t es, int64_t k) {
  return es == 2 ? __uint_as_float((uint32_t)reinterpret_cast<const uint16_t*>(vals)[k] << 16)
                 : __uint_as_float(reinterpret_cast<const uint32_t*>(vals)[k]);
}

// the sketch's w'(o, j) of a fast-path layout (ROW units, g = 1, raw states): unit j, position o
__device__ __forceinline__ float sketch_value_row(const QArgs& A, const QLayer& Ly, int64_t o, int64_t j) {
  const int64_t u = Ly.unit_base + j;
  const uint32_t N = (uint32_t)A.ncols[u];
  const int64_t off = A.offsets[u];
  const uint32_t Ku = A.ukeys[u];
  const int Mu = A.nrows[u];
  uint32_t best = 0;
  for (int i = 0; i < Mu; ++i) {
    const uint32_t idx = hash_index_x(A.hc, (uint32_t)o, Ku, i, N);
    const int64_t c = off + (int64_t)i * N + idx;
    const uint32_t b = A.es == 2 ? ((uint32_t)reinterpret_cast<const uint16_t*>(A.sketch)[c] << 16)
                                 : reinterpret_cast<const uint32_t*>(A.sketch)[c];
    best = max(best, rotl1(b) ^ 1u);
  }
  return __uint_as_float(rotr1(best) ^ 0x80000000u);
}

constexpr int kRedThreads = 256;

// y[r] = sum of row r's chunk partials in a fixed order: a group of red_lanes (power of two)
// lanes per row; lane j sums chunks [4j, 4j + 4) of every 4*red_lanes-chunk stride with one
// coalesced float4 load each, then an xor butterfly over the group (every lane ends with the same
// bits, so the result is deterministic).
__global__ void __launch_bounds__(kRedThreads, 8) k_gemv_reduce(const __grid_constant__ QArgs A) {
  if (A.timeline && threadIdx.x == 0) A.timeline[blockIdx.x * kTS + 0] = gtimer();
  pdl_trigger();  // the next call's compute kernel may be scheduled (it stages before its own wait)
  // every kernel-parameter read happens before the wait: a first touch of a parameter line misses
  // the SM's constant cache (~1 us), which would otherwise sit on the critical path
  const int L = A.red_lanes;
  const int64_t g = (int64_t)blockIdx.x * kRedThreads + threadIdx.x;
  const int64_t r = g / L;
  const int j = (int)(g % L);
  int li = 0;
  if (r < A.rows)
    while (li + 1 < A.n_layers && A.layer[li + 1].row_begin <= r) ++li;
  const QLayer& Ly = A.layer[li];
  const int64_t rr = r - Ly.row_begin;
  const int nch = Ly.n_chunks;
  const float4* p = reinterpret_cast<const float4*>(Ly.partial + rr * Ly.CP);
  void* const yp = Ly.y;
  const int64_t n_out = Ly.n_out;
  const bool y_bf16 = A.y_bf16 != 0;
  unsigned long long* const tl = A.timeline;
  asm volatile("" ::"l"(p), "l"(yp), "l"(n_out), "r"(nch), "r"((int)y_bf16), "l"(tl) : "memory");
  pdl_wait();     // all chunk partials written
  if (tl && threadIdx.x == 0) tl[blockIdx.x * kTS + 1] = gtimer();
  float t = 0.f;
  if (r < A.rows) {
    for (int c = 4 * j; c < nch; c += 4 * L) {
      const float4 q = __ldcg(p + c / 4);
      t += q.x;
      if (c + 1 < nch) t += q.y;
      if (c + 2 < nch) t += q.z;
      if (c + 3 < nch) t += q.w;
    }
  }
  for (int m = 1; m < L; m <<= 1) t += __shfl_xor_sync(0xffffffffu, t, m);
  if (r < A.rows && j == 0) {
    if (n_out) {  // Top-K: outliers contribute x_j * (w - w'_sketch) on top, in index order
      const int64_t o = Ly.o_begin + rr;
      int64_t lo, hi;
      outlier_range(Ly.oidx, Ly.n_out, o, A.in, lo, hi);
      float corr = 0.f;
      for (int64_t k = lo; k < hi; ++k) {
        const int64_t jj = (int64_t)(uint32_t)Ly.oidx[k] - o * A.in;
        const float xv = A.x_bf16 ? __uint_as_float((uint32_t)reinterpret_cast<const uint16_t*>(A.x)[jj] << 16)
                                  : reinterpret_cast<const float*>(A.x)[jj];
        corr = fmaf(xv, state_value(Ly.ovals, A.es, k) - sketch_value_row(A, Ly, o, jj), corr);
      }
      t += corr;
    }
    if (y_bf16) {
      const uint32_t bb = __float_as_uint(t);
      reinterpret_cast<uint16_t*>(yp)[rr] = (uint16_t)((bb + 0x7FFFu + ((bb >> 16) & 1u)) >> 16);
    } else {
      reinterpret_cast<float*>(yp)[rr] = t;
    }
  }
  if (tl && (threadIdx.x & 31) == 0) {
    atomicMax(&tl[blockIdx.x * kTS + 2], gtimer());
    atomicMax(&tl[blockIdx.x * kTS + 3], gtimer());
  }
}

// ------------------------------------------------------------------ generic query path
struct GenQ {
  const void* sketch;
  const int32_t* ncols;
  const uint8_t* nrows;   // M_u per unit (ledger L30)
  const int64_t* offsets;
  const uint32_t* ukeys;
  HashConsts hc;
  int64_t unit_base, out, in;
  int32_t M, gran, g, hash, es;
  int32_t q, g_shift;     // quantised plans (L25)
  const float* scales;
  int32_t variant;        // usk_variant (L27)
  const int32_t* oidx;    // Top-K side table, or NULL
  const void* ovals;
  int64_t n_out;
};

// cell value as fp32 bits (raw bf16: bits << 16; quantised: fl32(code * scale))
__device__ __forceinline__ uint32_t gen_cell_bits(const GenQ& Q, int64_t c) {
  if (Q.q == 0)
    return Q.es == 2 ? ((uint32_t)reinterpret_cast<const uint16_t*>(Q.sketch)[c] << 16)
                     : reinterpret_cast<const uint32_t*>(Q.sketch)[c];
  const uint8_t* codes = reinterpret_cast<const uint8_t*>(Q.sketch);
  int code;
  if (Q.q == 8) {
    code = (int)(int8_t)codes[c];
  } else {
    code = (int)((codes[c >> 1] >> ((c & 1) * 4)) & 0xFu);
    code = (code ^ 8) - 8;
  }
  return __float_as_uint(__fmul_rn((float)code, Q.scales[c >> Q.g_shift]));
}

__device__ __forceinline__ uint32_t gen_weight_bits_hi(const GenQ& Q, int64_t o, int64_t j) {
  int64_t t, p;
  unit_pos(Q.gran, Q.g, Q.out, o, j, t, p);
  const int64_t u = Q.unit_base + t;
  const uint32_t N = (uint32_t)Q.ncols[u];
  const int64_t off = Q.offsets[u];
  const uint32_t Ku = Q.ukeys[u];
  const int Mu = Q.nrows[u];
  if (Q.variant != USK_ABSMAXMIN) {
    // AbsMinMax / CountMin: the bonded cell of MINIMUM |.|, ties -> non-negative = min kappa
    uint32_t best = 0xFFFFFFFFu;
    for (int i = 0; i < Mu; ++i) {
      const uint32_t idx = Q.hash == USK_HASH_X ? hash_index_x(Q.hc, (uint32_t)p, Ku, i, N) : (uint32_t)(p % N);
      best = min(best, rotl1(gen_cell_bits(Q, off + (int64_t)i * N + idx)));
    }
    return rotr1(best);
  }
  uint32_t best = 0;
  for (int i = 0; i < Mu; ++i) {
    const uint32_t idx = Q.hash == USK_HASH_X ? hash_index_x(Q.hc, (uint32_t)p, Ku, i, N) : (uint32_t)(p % N);
    const int64_t c = off + (int64_t)i * N + idx;
    best = max(best, rotl1(gen_cell_bits(Q, c)) ^ 1u);
  }
  return rotr1(best) ^ 0x80000000u;
}

__global__ void k_reconstruct_gen(GenQ Q, int64_t o0, int64_t o1, void* w_out, int64_t ld) {
  const int64_t n = (o1 - o0) * Q.in;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / Q.in, j = e - r * Q.in;
    uint32_t b = gen_weight_bits_hi(Q, o0 + r, j);
    if (Q.es == 2 && Q.q) b = b + 0x7FFFu + ((b >> 16) & 1u);  // quantised: RNE to bf16
    if (Q.es == 2) reinterpret_cast<uint16_t*>(w_out)[r * ld + j] = (uint16_t)(b >> 16);
    else reinterpret_cast<uint32_t*>(w_out)[r * ld + j] = b;
  }
}

// Top-K overlay of the reconstruction (L29): rows [o0, o1) of w_out (ld) get the
// outliers' exact states
__global__ void k_overlay(const int32_t* idx, const void* vals, int64_t n, int32_t es, int64_t in, int64_t o0,
                          int64_t o1, void* w_out, int64_t ld) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int64_t e = (int64_t)(uint32_t)idx[k], o = e / in, j = e - o * in;
  if (o < o0 || o >= o1) return;
  if (es == 2) reinterpret_cast<uint16_t*>(w_out)[(o - o0) * ld + j] = reinterpret_cast<const uint16_t*>(vals)[k];
  else reinterpret_cast<uint32_t*>(w_out)[(o - o0) * ld + j] = reinterpret_cast<const uint32_t*>(vals)[k];
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
  if (lane == 0 && Q.n_out) {  // Top-K: outliers contribute x_j * (w - w'_sketch), in index order
    const int64_t o = o0 + r;
    int64_t lo, hi;
    outlier_range(Q.oidx, Q.n_out, o, Q.in, lo, hi);
    float corr = 0.f;
    for (int64_t k = lo; k < hi; ++k) {
      const int64_t jj = (int64_t)(uint32_t)Q.oidx[k] - o * Q.in;
      const float xv = x_bf16 ? __uint_as_float((uint32_t)reinterpret_cast<const uint16_t*>(x)[jj] << 16)
                              : reinterpret_cast<const float*>(x)[jj];
      corr = fmaf(xv, state_value(Q.ovals, Q.es, k) - __uint_as_float(gen_weight_bits_hi(Q, o, jj)), corr);
    }
    s += corr;
  }
  if (lane == 0) {
    if (y_bf16) {
      const uint32_t b = __float_as_uint(s);
      reinterpret_cast<uint16_t*>(y)[r] = (uint16_t)((b + 0x7FFFu + ((b >> 16) & 1u)) >> 16);
    } else {
      reinterpret_cast<float*>(y)[r] = s;
    }
  }
}

// ------------------------------------------------------------------ K7: compression report
// (SPEC stats; DESIGN.md ledger L27).  Integer counts with integer atomics: deterministic.
__global__ void k_stats_weights(GenQ Q, const void* W, unsigned long long* counts, int32_t* occ) {
  __shared__ unsigned int sc[11];
  if (threadIdx.x < 11) sc[threadIdx.x] = 0;
  __syncthreads();
  const int64_t n = Q.out * Q.in;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t o = e / Q.in, j = e - o * Q.in;
    uint32_t pb = gen_weight_bits_hi(Q, o, j);  // w' (fp32 bits; bf16 in the high half)
    if (Q.es == 2 && Q.q) pb = pb + 0x7FFFu + ((pb >> 16) & 1u);
    if (Q.n_out) {  // Top-K: outliers keep their value
      int64_t lo, hi;
      outlier_range(Q.oidx, Q.n_out, o, Q.in, lo, hi);
      for (int64_t k = lo; k < hi; ++k)
        if ((int64_t)(uint32_t)Q.oidx[k] == e) pb = __float_as_uint(state_value(Q.ovals, Q.es, k));
    }
    uint32_t wb;
    if (Q.es == 2) {
      wb = (uint32_t)reinterpret_cast<const uint16_t*>(W)[e] << 16;
      pb &= 0xFFFF0000u;
    } else {
      wb = reinterpret_cast<const uint32_t*>(W)[e];
    }
    const float w = __uint_as_float(wb), wp = __uint_as_float(pb);
    atomicAdd(&sc[0], 1u);
    if (wb == pb) atomicAdd(&sc[1], 1u);
    if (w != 0.f && wp != 0.f && ((wb ^ pb) & 0x80000000u)) atomicAdd(&sc[2], 1u);
    if (w == 0.f) {
      atomicAdd(&sc[3], 1u);
    } else {
      const float r = __fdiv_rn(fabsf(__fsub_rn(w, wp)), fabsf(w));
      int b = 0;
      if (r > 0.f) b = r < 1e-3f ? 1 : r < 1e-2f ? 2 : r < 1e-1f ? 3 : r < 1.f ? 4 : r < 10.f ? 5 : 6;
      atomicAdd(&sc[4 + b], 1u);
    }
    // occupancy: one count per sketch row
    int64_t t, p;
    unit_pos(Q.gran, Q.g, Q.out, o, j, t, p);
    const int64_t u = Q.unit_base + t;
    const uint32_t N = (uint32_t)Q.ncols[u];
    const uint32_t Ku = Q.ukeys[u];
    const int64_t base = Q.offsets[u] - Q.offsets[Q.unit_base];
    for (int i = 0; i < (int)Q.nrows[u]; ++i) {
      const uint32_t idx = Q.hash == USK_HASH_X ? hash_index_x(Q.hc, (uint32_t)p, Ku, i, N) : (uint32_t)(p % N);
      atomicAdd(&occ[base + (int64_t)i * N + idx], 1);
    }
  }
  __syncthreads();
  if (threadIdx.x < 11 && sc[threadIdx.x]) atomicAdd(&counts[threadIdx.x], (unsigned long long)sc[threadIdx.x]);
}

__global__ void k_stats_cells(int32_t* occ, int64_t n, unsigned long long* counts) {
  __shared__ unsigned int z;
  if (threadIdx.x == 0) z = 0;
  __syncthreads();
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c < n) {
    if (occ[c] == 0) atomicAdd(&z, 1u);
    occ[c] = 0;  // leave the workspace zeroed
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (z) atomicAdd(&counts[12], (unsigned long long)z);
    if (blockIdx.x == 0) atomicAdd(&counts[11], (unsigned long long)n);
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
bool fast_eligible(const usk_plan* pl) {
  return pl->gran == USK_GRAN_ROW && pl->g == 1 && pl->variant == USK_ABSMAXMIN;
}

constexpr size_t kSmemMax = 220 * 1024;

// raw staging bytes of `pu` units: cell bytes (raw plans) or packed codes (quantised, q bits);
// the staged scales follow at a 16-B aligned offset (quantised plans)
size_t raw_bytes(int maxMN, int es, int q, int pu) {
  return q ? ((size_t)pu * maxMN * q + 7) / 8 + 48 : (size_t)pu * maxMN * es + 48;
}
size_t sbuf_bytes(int maxMN, int q, int g_shift, int pu) {
  return q ? ((((size_t)pu * maxMN) >> g_shift) + 3) * 4 + 32 : 0;
}

// [zero + mbarrier + copy bases][rho cells][raw bulk-copy buffer for `pu` units][scales]
size_t smem_bytes(int upl, int maxMN, int es, int pu, int q = 0, int g_shift = 7) {
  return kCellsWordOffset * 4 + 128 + (size_t)32 * upl * maxMN * 4 + (raw_bytes(maxMN, es, q, pu) + 15) / 16 * 16 +
         sbuf_bytes(maxMN, q, g_shift, pu);
}

template <typename E, int UPL, bool GEMV, int QB, bool XB = false>
void* pick_m(int M, int hash) {
  if constexpr (GEMV) {
    if (hash == USK_HASH_IDENTITY) return (void*)k_gemv_fast<E, UPL, 0, USK_HASH_IDENTITY, QB, XB>;
    if constexpr (QB == 0) {
      switch (M) {
        case 1: return (void*)k_gemv_fast<E, UPL, 1, USK_HASH_X, QB, XB>;
        case 2: return (void*)k_gemv_fast<E, UPL, 2, USK_HASH_X, QB, XB>;
        default: break;
      }
    }
    return M == 3 ? (void*)k_gemv_fast<E, UPL, 3, USK_HASH_X, QB, XB> : (void*)k_gemv_fast<E, UPL, 0, USK_HASH_X, QB, XB>;
  } else {
    if (hash == USK_HASH_IDENTITY) return (void*)k_recon_fast<E, UPL, 0, USK_HASH_IDENTITY, QB>;
    if constexpr (QB == 0) {
      switch (M) {
        case 1: return (void*)k_recon_fast<E, UPL, 1, USK_HASH_X, QB>;
        case 2: return (void*)k_recon_fast<E, UPL, 2, USK_HASH_X, QB>;
        default: break;
      }
    }
    return M == 3 ? (void*)k_recon_fast<E, UPL, 3, USK_HASH_X, QB> : (void*)k_recon_fast<E, UPL, 0, USK_HASH_X, QB>;
  }
}

// quantised plans: the GEMV does not depend on the weight dtype (dequantised fp32 values, fp32 y),
// so only one E is instantiated for it; the reconstruct stores in the weight dtype.  Raw bf16 GEMVs
// with bf16 x multiply the key|value cells with fma.rn.f32.bf16 (XB).
template <int UPL, int QB>
void* pick_q(bool gemv, bool bf16, bool xbf16, int M, int hash) {
  if (gemv) {
    if constexpr (QB == 0) {
      if (!bf16) return pick_m<uint32_t, UPL, true, 0>(M, hash);
      return xbf16 ? pick_m<uint16_t, UPL, true, 0, true>(M, hash) : pick_m<uint16_t, UPL, true, 0, false>(M, hash);
    } else {
      return pick_m<uint32_t, UPL, true, QB>(M, hash);
    }
  }
  return bf16 ? pick_m<uint16_t, UPL, false, QB>(M, hash) : pick_m<uint32_t, UPL, false, QB>(M, hash);
}

template <int UPL>
void* pick_upl(bool gemv, bool bf16, bool xbf16, int M, int hash, int q) {
  switch (q) {
    case 4: return pick_q<UPL, 4>(gemv, bf16, xbf16, M, hash);
    case 8: return pick_q<UPL, 8>(gemv, bf16, xbf16, M, hash);
    default: return pick_q<UPL, 0>(gemv, bf16, xbf16, M, hash);
  }
}

void* pick_fast(int upl, bool gemv, bool bf16, bool xbf16, int M, int hash, int q) {
  switch (upl) {
    case 4: return pick_upl<4>(gemv, bf16, xbf16, M, hash, q);
    case 2: return pick_upl<2>(gemv, bf16, xbf16, M, hash, q);
    default: return pick_upl<1>(gemv, bf16, xbf16, M, hash, q);
  }
}

int ilog2(int v) {
  int r = 0;
  while ((1 << r) < v) ++r;
  return r;
}

int sm_count() { return device_sm_count(); }

int occupancy(void* kern, size_t smem) {
  // cached per (device, kernel, smem); the max-dynamic-smem attribute is raised per device on first
  // use (callers warm up before any graph capture)
  static std::mutex mu;
  static std::vector<std::pair<std::tuple<int, void*, size_t>, int>> cache;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    (void)cudaGetLastError();
    return 0;
  }
  const auto key = std::make_tuple(dev, kern, smem);
  {
    std::lock_guard<std::mutex> lock(mu);
    for (auto& e : cache)
      if (e.first == key) return e.second;
  }
  if (ensure_smem(kern, (int)kSmemMax) != cudaSuccess) return 0;
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kQThreads, smem) != cudaSuccess) {
    (void)cudaGetLastError();
    occ = 0;
  }
  std::lock_guard<std::mutex> lock(mu);
  cache.push_back({key, occ});
  return occ;
}

int env_int(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return e ? std::atoi(e) : dflt;
}

struct Geom {
  int upl = 0;
  int sub = kSubRows;  // rows per subtile item
  int maxMN = 0;
  int pu = 0;  // units per staging bulk copy
  size_t smem = 0;
  int grid = 0;
  void* kern = nullptr;
  int64_t items = 0;
  std::vector<int> n_chunks, n_sub;
};

// Query geometry (K3 and K4).  Units per lane: the largest UPL whose CTA fits the shared-memory
// budget (default 220 KB); the raw staging buffer shrinks to pieces of pu units before UPL does.
// Grid: one CTA per SM (USK_GEMV_CPS per SM for tuning), never more than the work items.
// USK_UPL / USK_GEMV_SMEM_KB / USK_GEMV_CPS override (tuning).
Geom gemv_geometry(const usk_plan* pl, const int32_t* layers, const int64_t* rows, int n, bool gemv = true,
                   bool xbf16 = false) {
  Geom G;
  for (int k = 0; k < n; ++k) G.maxMN = std::max(G.maxMN, pl->M * (pl->layers[layers[k]].max_ncols + 1));
  const int64_t in = pl->layers[layers[0]].in;
  const bool bf16 = pl->dtype == USK_BF16;
  const int es = pl->cell_bytes();
  static const int forced = env_int("USK_UPL", 0);
  static const size_t budget = (size_t)env_int("USK_GEMV_SMEM_KB", 220) * 1024;
  static const int cps = std::max(1, env_int("USK_GEMV_CPS", 1));
  for (int pass = 0; pass < 2 && !G.upl; ++pass) {  // pass 1: any fit below the hardware limit
    const size_t cap = pass == 0 ? std::min(budget, kSmemMax) : kSmemMax;
    for (int upl : {4, 2, 1}) {
      if (forced && upl != forced) continue;
      for (int pu = 32 * upl; pu >= 8; pu /= 2) {
        const size_t sm = smem_bytes(upl, G.maxMN, es, pu, pl->q, ilog2(pl->G));
        if (sm > cap) continue;
        void* kern = pick_fast(upl, gemv, bf16, xbf16, pl->M, pl->hash, pl->q);
        const int occ = occupancy(kern, sm);
        if (occ < 1) continue;
        G.upl = upl;
        G.pu = pu;
        G.smem = sm;
        G.kern = kern;
        G.grid = sm_count() * std::min(occ, cps);
        break;
      }
      if (G.upl) break;
    }
  }
  if (!G.upl) return G;
  // 8-row subtiles (raw bf16 GEMV with bf16 x, M = 3): when a CTA's share of 16-row items ends in a
  // mostly idle round of its 16 warps.  Estimated CTA time = rounds x item time, the 8-row loop
  // costing ~15 % more per weight in the product (in-graph trace: Llama-3.2-1B down, 3.5 items per
  // warp at 16 rows, mean compute 13.8 vs 12.8 us with 8 rows; the loop alone: 1792 vs 1898 G w/s).
  static const int forced_sub = env_int("USK_SUB", 0);
  auto items_at = [&](int sub) {
    int64_t it = 0;
    for (int k = 0; k < n; ++k) it += ((in + 32 * G.upl - 1) / (32 * G.upl)) * ((rows[k] + sub - 1) / sub);
    return it;
  };
  if (gemv && xbf16 && pl->dtype == USK_BF16 && pl->q == 0 && pl->M == 3 && pl->hash == USK_HASH_X && kSubRows == 16) {
    const int warps = kQThreads / 32;
    auto est = [&](int sub) {
      const int64_t it = items_at(sub);
      const int64_t ctas = std::min<int64_t>(G.grid, it);
      const double per = (double)it / (double)ctas;
      return std::ceil(per / warps) * sub * (sub == 8 ? 1.15 : 1.0);
    };
    const int want = forced_sub ? forced_sub : (est(8) < est(16) ? 8 : 16);
    if (want == 8 && G.upl == 4) {
      void* k8 = (void*)k_gemv_fast<uint16_t, 4, 3, USK_HASH_X, 0, true, 8>;
      if (occupancy(k8, G.smem) >= 1) {
        G.sub = 8;
        G.kern = k8;
      }
    }
  }
  for (int k = 0; k < n; ++k) {
    G.n_chunks.push_back((int)((in + 32 * G.upl - 1) / (32 * G.upl)));
    G.n_sub.push_back((int)((rows[k] + G.sub - 1) / G.sub));
    G.items += (int64_t)G.n_chunks.back() * G.n_sub.back();
  }
  G.grid = (int)std::min<int64_t>(G.grid, std::max<int64_t>(G.items, 1));
  return G;
}

int partial_stride(int64_t in) { return (int)((((in + 31) / 32) + 3) / 4 * 4); }

// per layer: [partials rows x CP floats][256 B control: grid-barrier counters]
size_t layer_ws_ctrl_off(int64_t in, int64_t rows) { return ((size_t)rows * partial_stride(in) * 4 + 255) / 256 * 256; }
size_t layer_ws_bytes(int64_t in, int64_t rows) { return layer_ws_ctrl_off(in, rows) + 256; }

// Top-K side table of layer l (L29) into a launch layer
void set_outliers(const usk_plan* pl, int32_t l, const void* sketch, QLayer& Ly) {
  const LayerGeom& L = pl->layers[l];
  Ly.n_out = L.n_out;
  Ly.out_rows = L.out;
  if (!L.n_out) return;
  const char* tab = reinterpret_cast<const char*>(sketch) + L.out_off;
  Ly.oidx = reinterpret_cast<const int32_t*>(tab);
  Ly.ovals = tab + (L.n_out * 4 + 15) / 16 * 16;
}

QArgs base_args(const usk_plan* pl, const void* sketch, int64_t in, const Geom& G) {
  QArgs A{};
  A.es = pl->cell_bytes();
  A.M = pl->M;
  A.maxMN = G.maxMN;
  A.maxN = G.maxMN / pl->M;
  A.row_bytes = 128u * (uint32_t)A.maxN;
  A.piece_units = G.pu;
  A.in = in;
  A.sketch = sketch;
  A.ncols = pl->d_ncols;
  A.nrows = pl->d_nrows;
  A.offsets = pl->d_offsets;
  A.ukeys = pl->d_keys;
  A.hc = pl->hc;
  if (pl->q) {
    A.g_shift = ilog2(pl->G);
    A.sbuf_off = (int32_t)((raw_bytes(G.maxMN, pl->cell_bytes(), pl->q, G.pu) + 15) / 16 * 16);
    A.scales = reinterpret_cast<const float*>(reinterpret_cast<const char*>(sketch) + pl->scales_off);
  }
  return A;
}

// Balanced CTA item ranges for k_gemv_fast.  Every chunk boundary inside a CTA's range costs P
// items of time (one more chunk staging + warp drain): P = 8 + (slot cells per chunk) / 1024
// items (fitted to the in-graph traces: ~40 for Llama-1B gate|up chunks, ~16 for the 2048-row
// layers; USK_SWITCH_ITEMS overrides).  Minimises the largest per-CTA cost over at most
// `G.grid` CTAs (binary search on the bound, greedy fill).  Fills A.cta_item, returns the grid.
int partition_items(QArgs& A, const Geom& G) {
  const int64_t I = A.items;
  const int cap = (int)std::min<int64_t>(std::min<int64_t>(G.grid, I), kMaxCtas);
  static const int forced_p = env_int("USK_SWITCH_ITEMS", -1);
  const int64_t P = (forced_p >= 0 ? forced_p : 8 + (int64_t)32 * G.upl * G.maxMN / 1024) * 16 / G.sub;  // in items
  auto chunk_end = [&](int64_t s) {
    int li = 0;
    while (li + 1 < A.n_layers && A.layer[li + 1].item_begin <= s) ++li;
    const QLayer& L = A.layer[li];
    return L.item_begin + ((s - L.item_begin) / L.n_sub + 1) * L.n_sub;
  };
  auto fill = [&](int64_t T, bool write) -> int {  // CTAs used (cap + 1: infeasible)
    int64_t pos = 0;
    int c = 0;
    while (pos < I) {
      if (c >= cap) return cap + 1;
      if (write) A.cta_item[c] = (int32_t)pos;
      int64_t budget = T, cur = pos;
      for (bool first = true; cur < I; first = false) {
        if (!first && (budget -= P) <= 0) break;
        const int64_t take = std::min(chunk_end(cur) - cur, budget);
        cur += take;
        budget -= take;
        if (budget <= 0) break;
      }
      pos = cur;
      ++c;
    }
    if (write) A.cta_item[c] = (int32_t)I;
    return c;
  };
  int64_t lo = (I + cap - 1) / cap, hi = lo;
  while (fill(hi, false) > cap) hi *= 2;
  while (lo < hi) {
    const int64_t mid = (lo + hi) / 2;
    if (fill(mid, false) <= cap) hi = mid;
    else lo = mid + 1;
  }
  return fill(lo, true);
}

// Raw plans: each CTA's first bulk copy (the first piece of the chunk at cta_item[c]) from the
// host copy of the unit offsets, the same bytes stage_issue would compute on the device.
void first_copies(const usk_plan* pl, QArgs& A, const Geom& G, int grid) {
  A.first_ok = 0;
  if (pl->q != 0) return;
  const int es = pl->cell_bytes();
  const int TJ = 32 * G.upl;
  for (int c = 0; c < grid; ++c) {
    const int64_t s = A.cta_item[c];
    if (s >= A.cta_item[c + 1]) {
      A.first_a0s[c] = 0;
      A.first_bytes[c] = 0;
      continue;
    }
    int li = 0;
    while (li + 1 < A.n_layers && A.layer[li + 1].item_begin <= s) ++li;
    const QLayer& L = A.layer[li];
    const int64_t chunk = (s - L.item_begin) / L.n_sub;
    const int64_t j0 = chunk * TJ;
    const int nu = (int)std::min<int64_t>(TJ, A.in - j0);
    const int pn = std::min(G.pu, nu);
    const int64_t ub = L.unit_base + j0;
    const uint64_t g0 = (uint64_t)pl->h_offsets[ub] * es, g1 = (uint64_t)pl->h_offsets[ub + pn] * es;
    const uint64_t a0 = g0 & ~uint64_t(15), a1 = (g1 + 15) & ~uint64_t(15);
    A.first_a0s[c] = a0 | (g0 - a0);
    A.first_bytes[c] = (uint32_t)(a1 - a0);
  }
  A.first_ok = 1;
}

// USK_TRACE (tuning only): per-CTA %globaltimer stamps of every query launch, slot per issue
struct Trace {
  static constexpr int64_t kCap = 1 << 18;  // CTAs
  std::mutex mu;
  bool on = std::getenv("USK_TRACE") != nullptr;
  unsigned long long* d = nullptr;
  int64_t cursor = 0;
  std::vector<int> grids;
};
Trace& trace() {
  static Trace T;
  return T;
}

// L2 warm-up (usk_prefetch_l2): up to 8 byte ranges; CTA c issues bulk L2 prefetches for its
// 1/grid slice of each (16-B granules), triggers the next launch at once, and waits for its own
// predecessor only after issuing (so stream order is kept transitively).  No data is returned.
struct PfRanges {
  const char* base[8];
  int64_t bytes[8];
  int32_t n;
};

__global__ void k_prefetch_l2(const __grid_constant__ PfRanges R) {
  if (threadIdx.x == 0)
    for (int r = 0; r < R.n; ++r) {
      const int64_t granules = R.bytes[r] >> 4;
      const int64_t per = (granules + gridDim.x - 1) / gridDim.x;
      const int64_t g0 = (int64_t)blockIdx.x * per, g1 = min(granules, g0 + per);
      for (int64_t g = g0; g < g1; g += 2048) {  // 32 KB per request
        const uint32_t n = (uint32_t)(min(g1 - g, (int64_t)2048) << 4);
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(R.base[r] + (g << 4)), "r"(n) : "memory");
      }
    }
  pdl_trigger();
  pdl_wait();
}

usk_status launch_prefetch_l2(const PfRanges& R, cudaStream_t st) {
  int64_t total = 0;
  for (int r = 0; r < R.n; ++r) total += R.bytes[r];
  if (total < 16) return USK_OK;
  const int grid = (int)std::min<int64_t>(sm_count(), (total + (256 << 10) - 1) / (256 << 10));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(32);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  USK_CUDA(cudaLaunchKernelEx(&cfg, k_prefetch_l2, R));
  count_launch();
  return USK_OK;
}

}  // namespace

// USK_TRACE (tuning only): the ring slot of a launch of `grid` CTAs (kTS stamps each), or nullptr
unsigned long long* trace_slot(int grid) {
  Trace& T = trace();
  std::lock_guard<std::mutex> lock(T.mu);
  if (!T.on) return nullptr;
  if (!T.d) {
    if (cudaMalloc(&T.d, sizeof(unsigned long long) * kTS * Trace::kCap) != cudaSuccess) return nullptr;
    if (cudaMemset(T.d, 0, sizeof(unsigned long long) * kTS * Trace::kCap) != cudaSuccess) return nullptr;
  }
  if (T.cursor + grid > Trace::kCap) T.cursor = 0, T.grids.clear();
  unsigned long long* p = T.d + kTS * T.cursor;
  T.cursor += grid;
  T.grids.push_back(grid);
  return p;
}

namespace {

usk_status launch_q(void* kern, const QArgs& A, int grid, size_t smem, bool pdl, cudaStream_t st,
                    int threads = kQThreads) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  QArgs B = A;
  {
    Trace& T = trace();
    std::lock_guard<std::mutex> lock(T.mu);
    if (T.on) {  // tuning only: stamps into this launch's slot of the ring
      if (!T.d) {
        USK_CUDA(cudaMalloc(&T.d, sizeof(unsigned long long) * kTS * Trace::kCap));
        USK_CUDA(cudaMemset(T.d, 0, sizeof(unsigned long long) * kTS * Trace::kCap));
      }
      if (T.cursor + grid > Trace::kCap) T.cursor = 0, T.grids.clear();
      B.timeline = T.d + kTS * T.cursor;
      T.cursor += grid;
      T.grids.push_back(grid);
    }
  }
  void* args[] = {&B};
  USK_CUDA(cudaLaunchKernelExC(&cfg, kern, args));
  count_launch();
  return USK_OK;
}

GenQ make_genq(const usk_plan* pl, int32_t l, const void* sketch) {
  const LayerGeom& L = pl->layers[l];
  GenQ Q{};
  Q.sketch = sketch;
  Q.ncols = pl->d_ncols;
  Q.nrows = pl->d_nrows;
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
  Q.q = pl->q;
  Q.g_shift = ilog2(pl->G);
  Q.scales = pl->q ? reinterpret_cast<const float*>(reinterpret_cast<const char*>(sketch) + pl->scales_off) : nullptr;
  Q.variant = pl->variant;
  Q.n_out = L.n_out;
  if (L.n_out) {
    const char* tab = reinterpret_cast<const char*>(sketch) + L.out_off;
    Q.oidx = reinterpret_cast<const int32_t*>(tab);
    Q.ovals = tab + (L.n_out * 4 + 15) / 16 * 16;
  }
  return Q;
}

}  // namespace

// usk_prefetch_l2: the sketch bytes of layers [a, b) -- raw cells, or the packed codes and the
// group scales of a quantised plan, plus the layers' Top-K side tables -- and the plan's per-unit
// metadata the query kernels read before their first cell (offsets, N_u, M_u, keys, classes)
usk_status launch_prefetch(const usk_plan* pl, const void* sketch, int32_t a, int32_t b, cudaStream_t st) {
  if (a >= b) return USK_OK;
  if (pl->layout == USK_LAYOUT_QUERY) {  // the layers' query-layout regions
    PfRanges R{};
    const int64_t lo = pl->layers[a].qoff, hi = pl->layers[b - 1].qoff + pl->layers[b - 1].qbytes;
    R.base[0] = reinterpret_cast<const char*>(sketch) + lo;
    R.bytes[0] = hi - lo;
    R.n = 1;
    return launch_prefetch_l2(R, st);
  }
  const LayerGeom& La = pl->layers[a];
  const LayerGeom& Lb = pl->layers[b - 1];
  const int64_t c0 = La.cell_begin, c1 = Lb.cell_begin + Lb.n_cells;
  const int64_t u0 = La.unit_begin, u1 = Lb.unit_begin + Lb.n_units;
  PfRanges R{};
  auto add = [&](const void* base, int64_t lo, int64_t hi) {
    lo &= ~int64_t(15);
    hi = (hi + 15) & ~int64_t(15);
    if (hi > lo && R.n < 8) {
      R.base[R.n] = reinterpret_cast<const char*>(base) + lo;
      R.bytes[R.n++] = hi - lo;
    }
  };
  if (pl->q == 0) {
    add(sketch, c0 * pl->cell_bytes(), c1 * pl->cell_bytes());
  } else {
    add(sketch, c0 * pl->q / 8, (c1 * pl->q + 7) / 8);
    add(sketch, pl->scales_off + c0 / pl->G * 4, pl->scales_off + (c1 + pl->G - 1) / pl->G * 4);
  }
  if (pl->side_bytes > 0 && La.n_out > 0) add(sketch, La.out_off, Lb.out_off + Lb.n_out * (4 + pl->cell_bytes()));
  // metadata arrays are allocated in whole 16-B granules? round inward at their ends to stay inside
  auto add_in = [&](const void* base, int64_t lo, int64_t hi) { add(base, lo, hi & ~int64_t(15)); };
  add_in(pl->d_offsets, u0 * 8, (u1 + 1) * 8);
  add_in(pl->d_ncols, u0 * 4, u1 * 4);
  add_in(pl->d_keys, u0 * 4, u1 * 4);
  add_in(pl->d_nrows, u0, u1);
  add_in(pl->d_cls, u0, u1);
  return launch_prefetch_l2(R, st);
}

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
  if (outrow_fast_ok(pl, layers, n))  // output-row units: one kernel, no split-K (outrow.cu)
    return launch_gemv_outrow(pl, sketch, layers, o0, o1, n, x, x_dtype, y, y_dtype, st);
  std::vector<int64_t> rows(n);
  for (int k = 0; k < n; ++k) rows[k] = o1[k] - o0[k];
  Geom G = fast_eligible(pl) ? gemv_geometry(pl, layers, rows.data(), n, true, x_dtype == USK_BF16) : Geom{};
  if (G.upl) {
    const int64_t in = pl->layers[layers[0]].in;
    QArgs A = base_args(pl, sketch, in, G);
    A.x = x;
    A.x_bf16 = x_dtype == USK_BF16;
    A.y_bf16 = y_dtype == USK_BF16;
    char* w = reinterpret_cast<char*>(ws);
    for (int k = 0; k < n; ++k) {
      if (rows[k] > 0) {
        QLayer& Ly = A.layer[A.n_layers++];
        Ly.unit_base = pl->layers[layers[k]].unit_begin;
        Ly.o_begin = o0[k];
        Ly.rows = rows[k];
        Ly.item_begin = A.items;
        Ly.row_begin = A.rows;
        Ly.n_chunks = G.n_chunks[k];
        Ly.n_sub = G.n_sub[k];
        Ly.CP = partial_stride(in);
        Ly.y = y[k];
        Ly.partial = reinterpret_cast<float*>(w);
        set_outliers(pl, layers[k], sketch, Ly);
        A.items += (int64_t)Ly.n_chunks * Ly.n_sub;
        A.rows += rows[k];
      }
      w += layer_ws_bytes(in, rows[k]);
    }
    if (!A.n_layers) return USK_OK;
    const int grid = partition_items(A, G);
    first_copies(pl, A, G, grid);
    A.red_lanes = 1;
    while (A.red_lanes < 32 && 4 * A.red_lanes < G.n_chunks[0]) A.red_lanes *= 2;
    usk_status s1 = launch_q(G.kern, A, grid, G.smem, true, st);
    if (s1 != USK_OK) return s1;
    // co-reside with k_gemv_fast's max-shared configuration (a hint: a failure is not an error)
    (void)ensure_func_attr((const void*)k_gemv_reduce, (int)cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    return launch_q((void*)k_gemv_reduce, A, (int)((A.rows * A.red_lanes + kRedThreads - 1) / kRedThreads), 0, true,
                    st, kRedThreads);
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
  Geom G = (fast_eligible(pl) && aligned) ? gemv_geometry(pl, &l, &rows, 1, false) : Geom{};
  if (G.upl) {
    QArgs A = base_args(pl, sketch, L.in, G);
    QLayer& Ly = A.layer[A.n_layers++];
    Ly.unit_base = L.unit_begin;
    Ly.o_begin = r0;
    Ly.rows = rows;
    Ly.item_begin = 0;
    Ly.n_chunks = G.n_chunks[0];
    Ly.n_sub = G.n_sub[0];
    Ly.w_out = w_out;
    Ly.ld_out = ld;
    A.items = (int64_t)Ly.n_chunks * Ly.n_sub;
    A.rows = rows;
    const int grid = partition_items(A, G);
    first_copies(pl, A, G, grid);
    // PDL: the kernel stages its sketch chunk (read-only) before griddepcontrol.wait and writes w_out
    // only after it, so it may start under the previous launch's tail (back-to-back reconstructs)
    usk_status s = launch_q(G.kern, A, grid, G.smem, true, st);
    if (s != USK_OK) return s;
  } else {
    GenQ Q = make_genq(pl, l, sketch);
    const int64_t n = rows * L.in;
    k_reconstruct_gen<<<(unsigned)std::min<int64_t>((n + 255) / 256, 148 * 16), 256, 0, st>>>(Q, r0, r1, w_out, ld);
    USK_LAUNCHED("k_reconstruct_gen");
  }
  if (L.n_out) {  // Top-K: the outliers keep their value (L29)
    const char* tab = reinterpret_cast<const char*>(sketch) + L.out_off;
    k_overlay<<<(unsigned)((L.n_out + 255) / 256), 256, 0, st>>>(reinterpret_cast<const int32_t*>(tab),
                                                                 tab + (L.n_out * 4 + 15) / 16 * 16, L.n_out,
                                                                 pl->cell_bytes(), L.in, r0, r1, w_out, ld);
    USK_LAUNCHED("k_overlay");
  }
  return USK_OK;
}

size_t stats_workspace_bytes(const usk_plan* pl, int32_t l) {
  return (size_t)std::max<int64_t>(pl->layers[l].n_cells, 1) * 4;
}

usk_status launch_stats(const usk_plan* pl, const void* sketch, int32_t l, const void* W, int64_t* counts, void* ws,
                        cudaStream_t st) {
  const LayerGeom& L = pl->layers[l];
  GenQ Q = make_genq(pl, l, sketch);
  unsigned long long* c = reinterpret_cast<unsigned long long*>(counts);
  USK_CUDA(cudaMemsetAsync(counts, 0, sizeof(int64_t) * USK_STATS_N, st));
  const int64_t n = L.out * L.in;
  k_stats_weights<<<(unsigned)std::min<int64_t>((n + 255) / 256, 148 * 16), 256, 0, st>>>(Q, W, c,
                                                                                           reinterpret_cast<int32_t*>(ws));
  USK_LAUNCHED("k_stats_weights");
  k_stats_cells<<<(unsigned)((std::max<int64_t>(L.n_cells, 1) + 255) / 256), 256, 0, st>>>(
      reinterpret_cast<int32_t*>(ws), L.n_cells, c);
  USK_LAUNCHED("k_stats_cells");
  return USK_OK;
}

usk_status launch_importance(const void* A, int32_t a_dtype, int64_t N, int64_t d, float* I, cudaStream_t st) {
  k_importance<<<(unsigned)((d + 255) / 256), 256, 0, st>>>(A, a_dtype == USK_BF16, N, d, I);
  USK_LAUNCHED("k_importance");
  return USK_OK;
}

}  // namespace usk

extern "C" {

size_t usk_stats_workspace_bytes(const usk_plan* pl, int32_t layer) {
  if (!pl || layer < 0 || layer >= pl->n_layers) return 0;
  return usk::stats_workspace_bytes(pl, layer);
}

usk_status usk_stats(const usk_plan* pl, const void* sketch, int32_t layer, const void* W, int64_t* counts,
                     void* workspace, size_t workspace_bytes, usk_stream stream) {
  if (!pl || !sketch || !W || !counts || !workspace) return usk::fail(USK_EINVAL, "usk_stats: null pointer");
  if (layer < 0 || layer >= pl->n_layers) return usk::fail(USK_ESHAPE, "usk_stats: layer out of range");
  if (workspace_bytes < usk::stats_workspace_bytes(pl, layer)) return usk::fail(USK_ESHAPE, "usk_stats: workspace");
  if (pl->layout != USK_LAYOUT_UNIT_MAJOR) return usk::fail(USK_EUNSUPPORTED, "usk_stats: unit-major layout only");
  return usk::launch_stats(pl, sketch, layer, W, counts, workspace, (cudaStream_t)stream);
}

int32_t usk_trace_read(uint64_t* stamps, int64_t cap_stamps, int32_t* grids, int32_t cap_launches) {
  usk::Trace& T = usk::trace();
  std::lock_guard<std::mutex> lock(T.mu);
  if (!T.on || !T.d) return 0;
  if (cudaDeviceSynchronize() != cudaSuccess) return 0;
  const int64_t n = std::min<int64_t>(usk::kTS * T.cursor, cap_stamps);
  if (stamps && n > 0 && cudaMemcpy(stamps, T.d, n * 8, cudaMemcpyDeviceToHost) != cudaSuccess) return 0;
  const int32_t nl = (int32_t)T.grids.size();
  for (int32_t k = 0; grids && k < std::min(nl, cap_launches); ++k) grids[k] = T.grids[k];
  return nl;
}

void usk_trace_reset(void) {
  usk::Trace& T = usk::trace();
  std::lock_guard<std::mutex> lock(T.mu);
  T.cursor = 0;
  T.grids.clear();
  if (T.d) (void)cudaMemset(T.d, 0, sizeof(unsigned long long) * usk::kTS * usk::Trace::kCap);
}

}  // extern "C"
