// packed.cu -- the query layout (usk.h USK_LAYOUT_QUERY; DESIGN.md §4, §5 "K4p", ledger L32).
//
// Query of one weight (Eq. 3 + Eq. 5; §3.1 decompress -> compute):
//   w'(o, j) = the bonded cell of maximum |.| over the M sketch rows (ties -> non-negative, L1/L2).
// Under USK-XG the 8 units (input dims) of a key group share the hash functions H_i (ledger L32), so
// for an output row o they read the SAME column idx_i(o) of their own cells.  The query layout puts
// those 8 cells side by side as 16-bit retrieve keys rho16 = rotl16(b, 1) ^ 1 (b = bf16 bits):
//
//   chunk = 256 units = 32 key groups (one per lane); slice (i, c) of a chunk = 32 x 16 B
//   byte ((i * maxN + c) * 32 + g) * 16 + 2 v  <-  cell (i, c) of unit 256 k + 8 g + v
//
// so a warp's gather of sketch row i for one output row is ONE ld.shared.v4 per lane (8 cells, four
// conflict-free 128-B wavefronts) instead of 8 scalar loads, the Eq. 5 max of two units is one
// VIMNMX3.U16x2 over the M = 3 rows, and the chunk is staged with one TMA bulk copy (no shared ->
// shared conversion: the layout IS the shared-memory layout).  The shared address of column idx is
// one FFMA.RZ with the result at ulp 512 (tests/test_oracle_hash.py::test_packed_float_form):
//   RZ(f * 512 N + (2^32 + B - 512 N)) = 2^32 + B + 512 idx,  f = 1 + (h mod 2^23) / 2^23
// and bits * 512 mod 2^32 = B + 512 idx: one IMAD adds the lane's 16 B.
//
// Kernels: k_qpack (unit-major cells -> query layout, build time), k_qgemv (decode, split-K over
// chunks, partials [rows][CP]) + k_qreduce (fixed-order sum, PDL-chained), k_qrecon (W' rows).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <mutex>
#include <tuple>
#include <vector>

#include "common.cuh"
#include "ptx.cuh"

namespace usk {
namespace {

#ifndef USK_QTHREADS
#define USK_QTHREADS 512
#endif
#ifndef USK_QMAXREG
#define USK_QMAXREG 112  // K4p / K3p (<= 96 used) + k_qreduce (256 x 32) share an SM's 64 K registers
#endif
constexpr int kPThreads = USK_QTHREADS;
constexpr int kPWarps = kPThreads / 32;
constexpr int kPSub = 16;          // output rows per warp work item (subtile)
constexpr int kPMaxLayers = 8;
constexpr int kPMaxCtas = 256;
constexpr int kPMaxM = 4;          // sketch rows of the query-layout kernels
constexpr int kPRedThreads = 256;
constexpr int kPHdr = 64;          // [2 mbarriers][s_next][pad]
constexpr int kPRtab = kPWarps * kPSub * 16;  // per warp: 16 rows x {R_0..R_3}
constexpr int kPTS = 8;            // USK_TRACE stamps per CTA
constexpr int kPZero = 1024;       // zero block before the slots (rows i >= M_k of a chunk, ledger L34)
constexpr int kPMaxPeers = 8;      // ranks of a fused y all-gather (one NVLink domain of B200s)

extern __shared__ __align__(16) unsigned char psm[];

struct PLayer {
  int64_t unit_base;   // global unit id of the layer's unit 0
  int64_t chunk0;      // global index of the layer's chunk 0 (d_qc_off / d_qc_N)
  int64_t o_begin;     // first output row of the launch range
  int64_t rows;
  int64_t item_begin;  // first work item (chunk-major, subtile-minor)
  int64_t row_begin;   // first row in the launch's reduction order
  int32_t n_chunks, n_sub, CP;
  int32_t st_al;       // reconstruct: ld_out and w_out allow 16-B row stores
  int32_t pc0;         // partial column of the entry's first chunk (entries are runs of one width)
  int32_t perm;        // chunk tables + qperm (class-ordered layers, ledger L34); else c * CW, M rows
  void* y;
  float* partial;      // [rows][CP]
  void* w_out;         // reconstruct
  int64_t ld_out;
};

struct PArgs {
  PLayer layer[kPMaxLayers];
  int32_t n_layers;
  int32_t nslot;        // staging slots (2: the next segment's bulk copy under this one's math)
  uint32_t slot_bytes;  // bytes per slot (max chunk bytes of the launch, 1024-aligned)
  int32_t y_bf16;
  int64_t in, items, rows;
  const unsigned char* sketch;
  const int64_t* qc_off;  // absolute byte offset of every chunk, [chunks + 1]
  const int32_t* qc_N;    // maxN of every chunk
  const int32_t* qc_q0;   // first query position (units, within the layer) of every chunk
  const int32_t* qc_n;    // units present in every chunk
  const int32_t* qc_M;    // sketch rows of every chunk (rows >= M_k read row 0: max unchanged)
  const int32_t* qperm;   // layer-local key group at each query position
  const int32_t* ncols;
  const uint32_t* ukeys;
  HashConsts hc;
  const void* x;
  int32_t red_lanes;
  int32_t n_ctas;       // compute CTAs of the launch
  int32_t x_prefetch;   // bulk L2 prefetch of the CTA's x slices before griddepcontrol.wait
  int32_t cta_item[kPMaxCtas + 1];
  uint64_t first_off[kPMaxCtas];   // CTA c's first bulk copy (host-computed: no dependent load)
  uint32_t first_bytes[kPMaxCtas];
  unsigned long long* timeline;    // tuning only (USK_TRACE)
  // fused y all-gather of an output-sharded decode (usk_linear_batch_peers): the reduce
  // kernel stores every row into the full y of each of the n_peers ranks (peer-mapped pointers), and
  // its last CTA raises this rank's flag in every rank's signal array to epoch + 1
  int32_t n_peers, my_rank;
  void* ypeer[kPMaxPeers][kPMaxLayers];  // [p][layer of the launch] -> rank p's full y of that layer
  uint32_t* sig[kPMaxPeers];             // rank p's signal array (uint32[n_peers])
  const uint32_t* epoch;                 // this rank's call counter (advanced by usk_peer_wait)
  unsigned int* done;                    // CTA arrival counter (workspace; left zero)
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ uint4 lds128(uint32_t a) {
  uint4 q;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(q.x), "=r"(q.y), "=r"(q.z), "=r"(q.w) : "r"(a));
  return q;
}
// the lane's UPL/2 words (UPL 16-bit cells) of one slice row: ld.shared.v4 (UPL 8), .v2 (UPL 4), .u32 (UPL 2)
template <int UPL>
__device__ __forceinline__ void lds_cells(uint32_t a, uint32_t (&w)[UPL / 2]) {
  if constexpr (UPL == 8) {
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(w[0]), "=r"(w[1 % (UPL / 2)]), "=r"(w[2 % (UPL / 2)]),
                 "=r"(w[3 % (UPL / 2)]) : "r"(a));
  } else if constexpr (UPL == 4) {
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(w[0]), "=r"(w[1 % (UPL / 2)]) : "r"(a));
  } else {
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(w[0]) : "r"(a));
  }
}
__device__ __forceinline__ uint32_t max_u16x2(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("max.u16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
// rotr16 of both halves of a pair of retrieve keys: the bf16 bits of -w' in each half
__device__ __forceinline__ uint32_t neg_w(uint32_t p) {
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, 0x7FFF7FFF, 0xE4;" : "=r"(d) : "r"(p >> 1), "r"(p << 15));
  return d;
}
// c + bf16 half of x * bf16 half of w (one FHFMA.BF16: exact product, one rounding)
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

// Row sums of an SR-row subtile (SR = 16, 8 or 4): acc[r] = this lane's partial of row r.  Every row
// is summed over the 32 lanes by ONE fixed tree whatever SR: lane bits 3, 2, 1, 0, then 4, each stage
// adding the partials of the two lanes across that bit (fp addition commutes, so both lanes of a
// pair agree).  With LS = 16 / SR, exchange-and-halve stages run on lane bits 3 .. log2(LS) (row
// bits SR/2 .. 1), plain butterflies on the lane bits below, then bit 4.  So a row's bits do not
// depend on SR (a per-launch choice), the output range, the batch or the GPU count (bit-identical
// shards).  The sum of row p_row<SR>(lane) is returned.
template <int SR>
__device__ __forceinline__ int p_row(int lane) { return (lane / (16 / SR)) & (SR - 1); }
template <int SR>
__device__ __forceinline__ bool p_writer(int lane) { return (lane & ((16 / SR - 1) | 16)) == 0; }

template <int SR>
__device__ __forceinline__ float transpose_reduce(float (&acc)[SR], int lane) {
  constexpr int LS = 16 / SR;
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
#pragma unroll
  for (int b = LS / 2; b >= 1; b >>= 1) t += __shfl_xor_sync(0xffffffffu, t, b);
  t += __shfl_xor_sync(0xffffffffu, t, 16);
  return t;
}

__device__ __forceinline__ uint64_t* p_bar(int s) { return reinterpret_cast<uint64_t*>(psm) + s; }
__device__ __forceinline__ int* p_next() { return reinterpret_cast<int*>(psm + 16); }
__device__ __forceinline__ uint32_t p_rtab() { return smem_u32(psm + kPHdr); }
// slots start 1024-B aligned (the ulp-512 address form needs B % 512 == 0)
// a 1024-B zero block (1024-aligned) precedes the slots: sketch rows a chunk does not have read it
__device__ __forceinline__ uint32_t p_zero() {
  const uint32_t a = smem_u32(psm + kPHdr + kPRtab);
  return (a + 1023u) & ~1023u;
}
template <bool TAB>
__device__ __forceinline__ uint32_t p_slot(const PArgs& A, int s) {
  return p_zero() + (TAB ? kPZero : 0u) + (uint32_t)s * A.slot_bytes;
}
template <bool TAB>
__device__ __forceinline__ void p_issue(const PArgs& A, int slot, uint64_t off, uint32_t bytes) {
  fence_proxy_async_smem();  // earlier generic reads of the slot happen before the async-proxy write
  mbar_arrive_expect_tx(p_bar(slot), bytes);
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   p_slot<TAB>(A, slot)),
               "l"(A.sketch + off), "r"(bytes), "r"(smem_u32(p_bar(slot)))
               : "memory");
}

struct PSeg {
  int li, chunk, sub_a, sub_end;
  int64_t end;
};

__device__ __forceinline__ PSeg p_seg_at(const PArgs& A, int64_t s, int64_t s_end) {
  PSeg g;
  g.li = 0;
  while (g.li + 1 < A.n_layers && A.layer[g.li + 1].item_begin <= s) ++g.li;
  const PLayer& L = A.layer[g.li];
  const int64_t local = s - L.item_begin;
  g.chunk = (int)(local / L.n_sub);
  g.sub_a = (int)(local - (int64_t)g.chunk * L.n_sub);
  g.end = min(s_end, L.item_begin + (int64_t)(g.chunk + 1) * L.n_sub);
  g.sub_end = g.sub_a + (int)(g.end - s);
  return g;
}

// Per-warp table of the subtile rows' position mixes R_i(o) mod 2^23 (rows past the range repeat
// the last row): lane r < 16 writes row r's {R_0..R_3}.
template <int MT, int SR>
__device__ __forceinline__ void p_fill_rtab(const PArgs& A, uint32_t rtab, int64_t o_first, int64_t o_last, int lane) {
  __syncwarp();
  if (lane < SR) {
    const uint32_t o = (uint32_t)min(o_first + lane, o_last);
    uint32_t r[4] = {0u, 0u, 0u, 0u};
#pragma unroll
    for (int i = 0; i < MT; ++i) r[i] = fmix32(o ^ A.hc.rho[i]) & 0x7FFFFFu;
    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(rtab + 16u * lane), "r"(r[0]), "r"(r[1]), "r"(r[2]),
                 "r"(r[3])
                 : "memory");
  }
  __syncwarp();
}

// K4p / K3p: one CTA per SM computes the host-balanced contiguous item range [cta_item[c],
// cta_item[c+1]) of (layer, chunk, 16-row subtile) items; warps grab the subtiles of a staged chunk.
// GEMV: chunk partials of every row -> [rows][CP].  !GEMV: W' rows (bf16) -> w_out.
template <int MT, bool GEMV, bool XB, int SR, int UPL, bool TAB>
__device__ __forceinline__ void p_query(const PArgs& A) {
  constexpr int CW = 32 * UPL;        // units per chunk (one lane's UPL units each)
  constexpr uint32_t SLB = 2u * CW;   // bytes per (sketch row, column) slice = the FFMA's ulp
  constexpr int PW = UPL / 2;         // 32-bit words (unit pairs) per lane and slice
  const int lane = threadIdx.x & 31;
  const int c = blockIdx.x;
  const int64_t s_begin = A.cta_item[c], s_end = A.cta_item[c + 1];
  unsigned long long* const tl = A.timeline ? A.timeline + (int64_t)c * kPTS : nullptr;
  if (tl && threadIdx.x == 0) tl[0] = gtimer();
  if (threadIdx.x == 0) {
    mbar_init(p_bar(0), 1);
    mbar_init(p_bar(1), 1);
    fence_mbar_init();
    if (s_begin < s_end) p_issue<TAB>(A, 0, A.first_off[c], A.first_bytes[c]);  // before anything else
    if (tl) tl[4] = gtimer();
  }
  if (TAB && threadIdx.x >= 64 && threadIdx.x < 64 + kPZero / 16)  // the zero block (read after the barrier below)
    asm volatile("st.shared.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(p_zero() + 16u * (threadIdx.x - 64)), "r"(0u)
                 : "memory");
  if (GEMV && A.x_prefetch && s_begin < s_end && threadIdx.x == 32) {
    // L2 warm-up of the x slices of this CTA's chunks (a pure hint: the loads after
    // griddepcontrol.wait read whatever the previous kernel wrote; L2 is the point of coherence)
    const int es = XB ? 2 : 4;
    int64_t s = s_begin;
    for (int n = 0; n < 4 && s < s_end; ++n) {
      const PSeg g = p_seg_at(A, s, s_end);
      const PLayer& Lp = A.layer[g.li];
      if (!TAB) {  // class-ordered chunks read x at scattered groups: no bulk hint
        const int64_t j0 = (int64_t)g.chunk * CW;
        const int64_t nb = min((int64_t)CW, A.in - j0) * es;
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(reinterpret_cast<const char*>(A.x) + j0 * es),
                     "r"((uint32_t)((nb + 15) & ~15ll))
                     : "memory");
      }
      s = g.end;
    }
  }
  bool waited = false;
  if (s_begin < s_end) {
    PSeg cur = p_seg_at(A, s_begin, s_end);
    if (threadIdx.x == 0) *p_next() = cur.sub_a;
    __syncthreads();  // mbarrier init + s_next visible
    uint32_t phase[2] = {0u, 0u};
    const uint32_t rtab = p_rtab() + (uint32_t)(threadIdx.x >> 5) * (kPSub * 16u);
    for (int k = 0;; ++k) {
      const int slot = A.nslot == 2 ? (k & 1) : 0;
      const PLayer& Ly = A.layer[cur.li];
      const bool more = cur.end < s_end;
      PSeg nxt = cur;
      if (more) nxt = p_seg_at(A, cur.end, s_end);
      // the other slot is free (its segment ended with a CTA barrier): next chunk's copy now
      if (A.nslot == 2 && more && threadIdx.x == 0) {
        const int64_t g = A.layer[nxt.li].chunk0 + nxt.chunk;
        const int64_t o0 = A.qc_off[g];
        p_issue<TAB>(A, slot ^ 1, (uint64_t)o0, (uint32_t)(A.qc_off[g + 1] - o0));
      }
      // lane state: units j0 .. j0 + UPL - 1 of the layer, inside one key group (they share K and N,
      // ledger L32; UPL 4 / 2: two / four lanes per group).  Chunk k holds query positions
      // q0_k .. q0_k + n_k - 1; a position is the unit itself, or (class-ordered layers, ledger L34)
      // unit 8 qperm[g0 + q / 8] + q % 8
      const int64_t gch = Ly.chunk0 + cur.chunk;
      int64_t j0;
      bool valid;
      int Mk = MT;
      if constexpr (!TAB) {  // identity order, one width: chunk c of the layer starts at unit c * CW, all rows
        j0 = (int64_t)cur.chunk * CW + UPL * lane;  // identity layers: one run, pc0 = 0
        valid = j0 < A.in;  // in % 8 == 0: a lane's units all exist or none
      } else {  // chunk tables (class-ordered layers, ledger L34; 64-unit chunks)
        const int qp = A.qc_q0[gch] + UPL * lane;
        valid = UPL * lane < A.qc_n[gch];
        j0 = valid ? 8 * (int64_t)A.qperm[(Ly.unit_base >> 3) + (qp >> 3)] + (qp & 7) : 0;  // unit_base % 8 == 0
        Mk = A.qc_M[gch];
      }
      const int64_t u0 = Ly.unit_base + j0;
      const uint32_t N = valid ? (uint32_t)A.ncols[u0] : 1u;
      const uint32_t K = valid ? A.ukeys[u0] : 0u;
      const uint32_t maxN = (uint32_t)A.qc_N[gch];
      const uint32_t B0 = p_slot<TAB>(A, slot);
      uint32_t fk[MT], cb[MT];
      float NS[TAB ? MT : 1];
#pragma unroll
      for (int i = 0; i < MT; ++i) {
        fk[i] = 0x3F800000u | (fmix32(K ^ A.hc.kap[i]) & 0x7FFFFFu);
        // SLB * 2^23 + B_i - SLB * N (a multiple of SLB in [SLB 2^22, SLB 2^24): an fp32 number); the
        // FFMA.RZ result lies at ulp SLB and bits * SLB mod 2^32 = B_i + SLB * idx + (exp << 23) * SLB
        // (biased exponent 159 / 158 / 157 for SLB 512 / 256 / 128: the last term wraps to 0, 0, 2^30;
        // LB removes it).  Sketch rows i >= M_k of the chunk (fewer rows than the kernel's): NS = 0 and
        // the FFMA returns SLB * 2^23 + Z exactly -- the zero block, neutral for the max.
        const bool row = !TAB || i < Mk;
        NS[TAB ? i : 0] = row ? (float)(SLB * N) : 0.f;
        cb[i] = __float_as_uint(__ull2float_rz(
            (unsigned long long)SLB * 8388608ull +
            (row ? B0 + (unsigned long long)i * maxN * SLB - (unsigned long long)SLB * N : p_zero())));
      }
      constexpr uint32_t EXPB = 127u + 23u + (SLB == 512u ? 9u : SLB == 256u ? 8u : 7u);
      const uint32_t LB = 2u * UPL * (uint32_t)lane - (EXPB << 23) * SLB;
      mbar_wait(p_bar(slot), phase[slot]);
      phase[slot] ^= 1u;
      if (!waited) {
        if (tl && threadIdx.x == 0) tl[5] = tl[6] = gtimer();
        if (GEMV) pdl_wait();  // x may be written by the previous kernel on the stream
        else pdl_wait();       // w_out may be read by the previous kernel
        pdl_trigger();
        if (tl && threadIdx.x == 0) tl[7] = gtimer();
        waited = true;
      }
      // -x of the lane's UPL inputs (bf16 pairs: sign bits flipped; fp32: negated)
      uint32_t nxb[PW];
      float nxf[UPL];
#pragma unroll
      for (int p = 0; p < PW; ++p) nxb[p] = 0u;
#pragma unroll
      for (int v = 0; v < UPL; ++v) nxf[v] = 0.f;
      if (GEMV && valid) {
        if constexpr (XB) {
          if constexpr (UPL == 8) {
            const uint4 xv = *reinterpret_cast<const uint4*>(reinterpret_cast<const uint16_t*>(A.x) + j0);
            nxb[0] = xv.x ^ 0x80008000u;
            nxb[1 % PW] = xv.y ^ 0x80008000u;
            nxb[2 % PW] = xv.z ^ 0x80008000u;
            nxb[3 % PW] = xv.w ^ 0x80008000u;
          } else if constexpr (UPL == 4) {
            const uint2 xv = *reinterpret_cast<const uint2*>(reinterpret_cast<const uint16_t*>(A.x) + j0);
            nxb[0] = xv.x ^ 0x80008000u;
            nxb[1 % PW] = xv.y ^ 0x80008000u;
          } else {
            nxb[0] = *reinterpret_cast<const uint32_t*>(reinterpret_cast<const uint16_t*>(A.x) + j0) ^ 0x80008000u;
          }
        } else if constexpr (UPL >= 4) {
#pragma unroll
          for (int q = 0; q < UPL / 4; ++q) {
            const float4 a = *reinterpret_cast<const float4*>(reinterpret_cast<const float*>(A.x) + j0 + 4 * q);
            nxf[4 * q] = -a.x, nxf[4 * q + 1] = -a.y, nxf[4 * q + 2] = -a.z, nxf[4 * q + 3] = -a.w;
          }
        } else {
          const float2 a = *reinterpret_cast<const float2*>(reinterpret_cast<const float*>(A.x) + j0);
          nxf[0] = -a.x, nxf[1 % UPL] = -a.y;
        }
      }
      if (tl && threadIdx.x == 0 && k == 0) tl[1] = gtimer();
      auto grab = [&]() -> int {
        int g = 0;
        if (lane == 0) g = atomicAdd(p_next(), 1);
        return __shfl_sync(0xffffffffu, g, 0);
      };
      int sub = grab();
      if (sub < cur.sub_end) p_fill_rtab<MT, SR>(A, rtab, Ly.o_begin + (int64_t)sub * SR, Ly.o_begin + Ly.rows - 1, lane);
      while (sub < cur.sub_end) {
        const int nsub = grab();  // issued now, consumed after this subtile
        const int64_t r0 = (int64_t)sub * SR;
        const int nrow = (int)min((int64_t)SR, Ly.rows - r0);
        if constexpr (GEMV) {
          float acc[SR];
#pragma unroll
          for (int r = 0; r < SR; ++r) {
            const uint4 R = lds128(rtab + 16u * r);
            const uint32_t Rv[4] = {R.x, R.y, R.z, R.w};
            uint32_t cl[MT][PW];
#pragma unroll
            for (int i = 0; i < MT; ++i) {
              const uint32_t bits =
                  __float_as_uint(__fmaf_rz(__uint_as_float(Rv[i] ^ fk[i]), NS[TAB ? i : 0], __uint_as_float(cb[i])));
              lds_cells<UPL>(bits * SLB + LB, cl[i]);
            }
            float a = 0.f;  // the lane's units in order
#pragma unroll
            for (int p = 0; p < PW; ++p) {
              uint32_t m = cl[0][p];
#pragma unroll
              for (int i = 1; i < MT; ++i) m = max_u16x2(m, cl[i][p]);
              const uint32_t wp = neg_w(m);
              if constexpr (XB) {
                a = fma_lo(nxb[p], wp, a);
                a = fma_hi(nxb[p], wp, a);
              } else {
                a = fmaf(nxf[2 * p], __uint_as_float(wp << 16), a);
                a = fmaf(nxf[2 * p + 1], __uint_as_float(wp & 0xFFFF0000u), a);
              }
            }
            acc[r] = a;
          }
          const float t = transpose_reduce<SR>(acc, lane);
          const int rr = p_row<SR>(lane);
          if (p_writer<SR>(lane) && rr < nrow) Ly.partial[(r0 + rr) * Ly.CP + (TAB ? Ly.pc0 : 0) + cur.chunk] = t;
        } else {
          uint16_t* dst = reinterpret_cast<uint16_t*>(Ly.w_out) + r0 * Ly.ld_out + j0;
#pragma unroll 4
          for (int r = 0; r < SR; ++r, dst += Ly.ld_out) {
            if (r >= nrow) break;
            const uint4 R = lds128(rtab + 16u * r);
            const uint32_t Rv[4] = {R.x, R.y, R.z, R.w};
            uint32_t cl[MT][PW];
#pragma unroll
            for (int i = 0; i < MT; ++i) {
              const uint32_t bits =
                  __float_as_uint(__fmaf_rz(__uint_as_float(Rv[i] ^ fk[i]), NS[TAB ? i : 0], __uint_as_float(cb[i])));
              lds_cells<UPL>(bits * SLB + LB, cl[i]);
            }
            // bits of w' = rotr16(rho) with the sign flipped back
            uint32_t w[PW];
#pragma unroll
            for (int p = 0; p < PW; ++p) {
              uint32_t m = cl[0][p];
#pragma unroll
              for (int i = 1; i < MT; ++i) m = max_u16x2(m, cl[i][p]);
              w[p] = neg_w(m) ^ 0x80008000u;
            }
            if (valid) {
              if (Ly.st_al) {
                if constexpr (UPL == 8) *reinterpret_cast<uint4*>(dst) = make_uint4(w[0], w[1 % PW], w[2 % PW], w[3 % PW]);
                else if constexpr (UPL == 4) *reinterpret_cast<uint2*>(dst) = make_uint2(w[0], w[1 % PW]);
                else *reinterpret_cast<uint32_t*>(dst) = w[0];
              } else {
#pragma unroll
                for (int v = 0; v < UPL; ++v) dst[v] = (uint16_t)(w[v >> 1] >> (16 * (v & 1)));
              }
            }
          }
        }
        sub = nsub;
        if (sub < cur.sub_end) p_fill_rtab<MT, SR>(A, rtab, Ly.o_begin + (int64_t)sub * SR, Ly.o_begin + Ly.rows - 1, lane);
      }
      __syncthreads();  // the slot and s_next are reused
      if (!more) break;
      if (threadIdx.x == 0) {
        *p_next() = nxt.sub_a;
        if (A.nslot == 1) {
          const int64_t g = A.layer[nxt.li].chunk0 + nxt.chunk;
          const int64_t o0 = A.qc_off[g];
          p_issue<TAB>(A, 0, (uint64_t)o0, (uint32_t)(A.qc_off[g + 1] - o0));
        }
      }
      __syncthreads();
      cur = nxt;
    }
  }
  if (!waited) {
    pdl_wait();
    pdl_trigger();
  }
  if (tl && lane == 0) {
    atomicMax(&tl[2], gtimer());
    atomicMax(&tl[3], gtimer());
  }
}

template <int MT, bool XB, int SR, int UPL, bool TAB>
__global__ void __maxnreg__(USK_QMAXREG) k_qgemv(const __grid_constant__ PArgs A) {
  p_query<MT, true, XB, SR, UPL, TAB>(A);
}

template <int MT, int UPL, bool TAB>
__global__ void __maxnreg__(USK_QMAXREG) k_qrecon(const __grid_constant__ PArgs A) {
  p_query<MT, false, false, 16, UPL, TAB>(A);
}

// y[r] = the fixed-order sum of row r's chunk partials: red_lanes lanes per row, lane j sums chunks
// [4j, 4j + 4) of every 4 * red_lanes stride (one float4 load each), then an xor butterfly (all lanes
// end with the same bits).  Launched with PDL: it waits for the partials, and triggers at once so the
// NEXT call's compute kernel stages its chunk while this one reduces.
__global__ void __launch_bounds__(kPRedThreads, 8) k_qreduce(const __grid_constant__ PArgs A) {
  unsigned long long* const tl = A.timeline ? A.timeline + (int64_t)blockIdx.x * kPTS : nullptr;
  if (tl && threadIdx.x == 0) tl[0] = gtimer();
  pdl_trigger();
  const int L = A.red_lanes;
  const int64_t g = (int64_t)blockIdx.x * kPRedThreads + threadIdx.x;
  const int64_t r = g / L;
  const int j = (int)(g % L);
  int li = 0;
  if (r < A.rows)
    while (li + 1 < A.n_layers && A.layer[li + 1].row_begin <= r) ++li;
  const PLayer& Ly = A.layer[li];
  const int64_t rr = r - Ly.row_begin;
  const int nch = Ly.n_chunks;
  const float4* p = reinterpret_cast<const float4*>(Ly.partial + rr * Ly.CP);
  void* const yp = Ly.y;
  const bool y_bf16 = A.y_bf16 != 0;
  asm volatile("" ::"l"(p), "l"(yp), "r"(nch), "r"((int)y_bf16) : "memory");
  pdl_wait();  // all chunk partials written (the compute grid completed)
  if (tl && threadIdx.x == 0) tl[1] = gtimer();
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
    const uint32_t bb = __float_as_uint(t);
    const uint16_t hb = (uint16_t)((bb + 0x7FFFu + ((bb >> 16) & 1u)) >> 16);
    if (A.n_peers == 0) {
      if (y_bf16) reinterpret_cast<uint16_t*>(yp)[rr] = hb;
      else reinterpret_cast<float*>(yp)[rr] = t;
    } else {  // the row at its global position in every rank's full y (NVLink peer stores)
      const int64_t o = Ly.o_begin + rr;
      for (int q = 0; q < A.n_peers; ++q) {
        void* yq = A.ypeer[q][li];
        if (y_bf16) reinterpret_cast<uint16_t*>(yq)[o] = hb;
        else reinterpret_cast<float*>(yq)[o] = t;
      }
    }
  }
  if (A.n_peers) {
    // publish: every CTA's peer stores are system-visible before its arrival; the last CTA to arrive
    // (it observed every arrival) raises this rank's flag in each rank's signal array
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned int prev = atomicAdd(A.done, 1u);
      if (prev == gridDim.x - 1) {
        __threadfence_system();
        const uint32_t e = *reinterpret_cast<const volatile uint32_t*>(A.epoch) + 1u;
        for (int q = 0; q < A.n_peers; ++q)
          asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(A.sig[q] + A.my_rank), "r"(e) : "memory");
        *A.done = 0u;
      }
    }
  }
  if (tl && (threadIdx.x & 31) == 0) {
    atomicMax(&tl[2], gtimer());
    atomicMax(&tl[3], gtimer());
  }
}

// usk_peer_wait: thread q < n_peers spins (acquire, system scope) until rank q's flag in this rank's
// signal array reaches epoch + 1, then the epoch advances.  Bounded: a peer that never signals leaves
// the flag short and sets err (reported by usk_check) instead of hanging the GPU.
__global__ void k_peer_wait(const uint32_t* sig, int32_t n_peers, uint32_t* epoch, int* err) {
  pdl_wait();
  const uint32_t want = *reinterpret_cast<const volatile uint32_t*>(epoch) + 1u;
  bool ok = true;
  if ((int)threadIdx.x < n_peers) {
    uint32_t v = 0;
    for (long spin = 0;; ++spin) {
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(sig + threadIdx.x) : "memory");
      if ((int32_t)(v - want) >= 0) break;
      if (spin > (1L << 24)) {
        ok = false;
        break;
      }
      __nanosleep(64);
    }
  }
  if (!ok) atomicOr(err, 4);  // a peer never signalled (usk_check: USK_ECUDA)
  __syncthreads();
  if (threadIdx.x == 0) *epoch = want;
  pdl_trigger();
}

// Unit-major cells -> query layout, one thread per 16-byte word (8 cells of a key group).  `ranges`:
// byte ranges [lo, hi) of the query sketch to write (whole chunks of the requested layers).
struct PackRanges {
  int64_t lo[16], hi[16], pre[17];  // pre: prefix of the ranges' 16-B word counts
  int32_t n;
};

__global__ void k_qpack(const __grid_constant__ PackRanges R, const uint16_t* __restrict__ cells,
                        const int64_t* __restrict__ qc_off, const int32_t* __restrict__ qc_N,
                        const int64_t* __restrict__ qc_ub, const int64_t* __restrict__ qc_g0,
                        const int32_t* __restrict__ qc_aux, const int32_t* __restrict__ qperm,
                        const int64_t* __restrict__ offsets, const int32_t* __restrict__ ncols,
                        const uint8_t* __restrict__ nrows, int64_t n_chunks, uint4* __restrict__ out) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= R.pre[R.n]) return;
  int r = 0;
  while (r + 1 < R.n && R.pre[r + 1] <= e) ++r;
  const int64_t byte = R.lo[r] + (e - R.pre[r]) * 16;
  int64_t a = 0, b = n_chunks;  // chunk: qc_off[a] <= byte < qc_off[a + 1]
  while (b - a > 1) {
    const int64_t m = (a + b) >> 1;
    if (qc_off[m] <= byte) a = m;
    else b = m;
  }
  const int64_t local = byte - qc_off[a];
  const int32_t maxN = qc_N[a];
  const int q0 = qc_aux[a], nu = qc_aux[n_chunks + a], Mk = qc_aux[2 * n_chunks + a], cw = qc_aux[3 * n_chunks + a];
  const int64_t slice = local / (2 * cw);  // slices of 2 * cw bytes, 8 units per 16-B word
  const int g = (int)((local % (2 * cw)) / 16);
  const int i = (int)(slice / maxN), col = (int)(slice % maxN);
  uint32_t w[4] = {0u, 0u, 0u, 0u};
#pragma unroll
  for (int v = 0; v < kQGroup; ++v) {
    const int s = g * kQGroup + v;  // slot in the chunk
    uint32_t key = 0u;
    if (s < nu && i < Mk) {
      const int qp = q0 + s;  // query position in the layer -> unit (class order: ledger L34)
      const int64_t u = qc_ub[a] + (qc_g0[a] >= 0 ? 8 * (int64_t)qperm[qc_g0[a] + (qp >> 3)] + (qp & 7) : (int64_t)qp);
      const int32_t N = ncols[u];
      if (col < N && i < (int)nrows[u]) {
        const uint32_t bb = cells[offsets[u] + (int64_t)i * N + col];
        key = ((((bb << 1) | (bb >> 15)) & 0xFFFFu) ^ 1u);
      }
    }
    w[v >> 1] |= key << (16 * (v & 1));
  }
  out[byte / 16] = make_uint4(w[0], w[1], w[2], w[3]);
}

// --------------------------------------------------------------------------------- host
int env_int(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return e ? std::atoi(e) : dflt;
}

int p_occupancy(const void* kern, size_t smem) {
  static std::mutex mu;
  static std::vector<std::pair<std::tuple<int, const void*, size_t>, int>> cache;
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
  if (ensure_smem(kern, 227 * 1024) != cudaSuccess) return 0;
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kPThreads, smem) != cudaSuccess) {
    (void)cudaGetLastError();
    occ = 0;
  }
  std::lock_guard<std::mutex> lock(mu);
  cache.push_back({key, occ});
  return occ;
}

template <int SR, int UPL, bool TAB>
const void* pick_gemv(bool xb, int M) {
  if (xb) {
    switch (M) {
      case 1: return (const void*)k_qgemv<1, true, SR, UPL, TAB>;
      case 2: return (const void*)k_qgemv<2, true, SR, UPL, TAB>;
      case 3: return (const void*)k_qgemv<3, true, SR, UPL, TAB>;
      default: return (const void*)k_qgemv<4, true, SR, UPL, TAB>;
    }
  }
  switch (M) {
    case 1: return (const void*)k_qgemv<1, false, SR, UPL, TAB>;
    case 2: return (const void*)k_qgemv<2, false, SR, UPL, TAB>;
    case 3: return (const void*)k_qgemv<3, false, SR, UPL, TAB>;
    default: return (const void*)k_qgemv<4, false, SR, UPL, TAB>;
  }
}

template <int UPL, bool TAB>
const void* pick_recon(int M) {
  switch (M) {
    case 1: return (const void*)k_qrecon<1, UPL, TAB>;
    case 2: return (const void*)k_qrecon<2, UPL, TAB>;
    case 3: return (const void*)k_qrecon<3, UPL, TAB>;
    default: return (const void*)k_qrecon<4, UPL, TAB>;
  }
}

// UPL: units per lane of the chunk width (cw = 32 * UPL: 256 -> 8, 128 -> 4, 64 -> 2).  tab: the
// launch has class-ordered layers (ledger L34) or 64-unit chunks -- the kernels read the chunk tables;
// identity-ordered launches compile without them (16- and 8-row subtiles only for tab)
const void* pick_kernel(bool gemv, bool xb, int M, int SR, int upl, bool tab) {
  if (gemv) {
    if (tab || upl == 2) {
      if (upl == 8) return SR == 16 ? pick_gemv<16, 8, true>(xb, M) : pick_gemv<8, 8, true>(xb, M);
      if (upl == 4) return SR == 16 ? pick_gemv<16, 4, true>(xb, M) : pick_gemv<8, 4, true>(xb, M);
      return SR == 16 ? pick_gemv<16, 2, true>(xb, M) : pick_gemv<8, 2, true>(xb, M);
    }
    if (upl == 8)
      return SR == 4 ? pick_gemv<4, 8, false>(xb, M) : SR == 8 ? pick_gemv<8, 8, false>(xb, M) : pick_gemv<16, 8, false>(xb, M);
    return SR == 4 ? pick_gemv<4, 4, false>(xb, M) : SR == 8 ? pick_gemv<8, 4, false>(xb, M) : pick_gemv<16, 4, false>(xb, M);
  }
  if (tab || upl == 2) return upl == 8 ? pick_recon<8, true>(M) : upl == 4 ? pick_recon<4, true>(M) : pick_recon<2, true>(M);
  return upl == 8 ? pick_recon<8, false>(M) : pick_recon<4, false>(M);
}

int partial_stride(int n_chunks) { return (n_chunks + 3) / 4 * 4; }
size_t layer_ws_bytes(int n_chunks, int64_t rows) { return ((size_t)rows * partial_stride(n_chunks) * 4 + 255) / 256 * 256; }

// Balanced CTA item ranges: minimise the largest per-CTA cost (items + P per chunk boundary inside
// a range: one more bulk copy and warp drain) over at most `cap` CTAs (binary search, greedy fill).
int p_partition(PArgs& A, int cap, int64_t P) {
  const int64_t I = A.items;
  cap = (int)std::min<int64_t>(std::min<int64_t>(cap, I), kPMaxCtas);
  auto chunk_end = [&](int64_t s) {
    int li = 0;
    while (li + 1 < A.n_layers && A.layer[li + 1].item_begin <= s) ++li;
    const PLayer& L = A.layer[li];
    return L.item_begin + ((s - L.item_begin) / L.n_sub + 1) * L.n_sub;
  };
  auto fill = [&](int64_t T, bool write) -> int {
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



usk_status p_launch(const void* kern, const PArgs& A, int grid, int threads, size_t smem, cudaStream_t st) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3((unsigned)threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  void* args[] = {const_cast<PArgs*>(&A)};
  USK_CUDA(cudaLaunchKernelExC(&cfg, kern, args));
  count_launch();
  return USK_OK;
}

// Query launch geometry shared by K4p and K3p: items, slots, partition, first copies.
usk_status p_prepare(const usk_plan* pl, PArgs& A, const void* kern, bool gemv, int& grid, size_t& smem, int sr = 16,
                     bool tab = false) {
  uint32_t slot = 0;
  for (int k = 0; k < A.n_layers; ++k) {
    const PLayer& L = A.layer[k];
    for (int c = 0; c < L.n_chunks; ++c)
      slot = std::max<uint32_t>(slot, (uint32_t)(pl->h_qc_off[L.chunk0 + c + 1] - pl->h_qc_off[L.chunk0 + c]));
  }
  slot = (slot + 1023u) & ~1023u;
  const size_t base = kPHdr + kPRtab + 1024 + (tab ? kPZero : 0);
  static const size_t cap = (size_t)env_int("USK_QSMEM_KB", 227) * 1024;
  static const int force_slots = env_int("USK_QSLOTS", 0);
  A.nslot = (base + 2 * (size_t)slot <= cap && force_slots != 1) ? 2 : 1;
  if (base + slot > 227 * 1024) return fail(USK_EUNSUPPORTED, "query layout: a chunk exceeds shared memory");
  A.slot_bytes = slot;
  smem = base + (size_t)A.nslot * slot;
  if (p_occupancy(kern, smem) < 1) return fail(USK_ECUDA, "query kernel does not fit an SM");
  // chunk-switch penalty in 16-row items (one more bulk copy + drain): 14 measured best on the 1B step
  // (2069 tok/s vs 2057 with 8 + slot / 16 KB, 1934 at 4, 1991 at 28; same box, interleaved)
  const int64_t P = (int64_t)env_int("USK_QSWITCH", 14) * 16 / sr;
  grid = p_partition(A, device_sm_count(), P);
  for (int c = 0; c < grid; ++c) {
    const int64_t s = A.cta_item[c];
    A.first_off[c] = 0;
    A.first_bytes[c] = 0;
    if (s >= A.cta_item[c + 1]) continue;
    int li = 0;
    while (li + 1 < A.n_layers && A.layer[li + 1].item_begin <= s) ++li;
    const PLayer& L = A.layer[li];
    const int64_t g = L.chunk0 + (s - L.item_begin) / L.n_sub;
    A.first_off[c] = (uint64_t)pl->h_qc_off[g];
    A.first_bytes[c] = (uint32_t)(pl->h_qc_off[g + 1] - pl->h_qc_off[g]);
  }
  (void)gemv;
  A.timeline = trace_slot(grid);
  return USK_OK;
}

PArgs p_base(const usk_plan* pl, const void* sketch, int64_t in) {
  PArgs A{};
  A.in = in;
  A.sketch = reinterpret_cast<const unsigned char*>(sketch);
  A.qc_off = pl->d_qc_off;
  A.qc_N = pl->d_qc_N;
  const size_t nch = pl->h_qc_N.size();
  A.qc_q0 = pl->d_qc_aux;
  A.qc_n = pl->d_qc_aux + nch;
  A.qc_M = pl->d_qc_aux + 2 * nch;
  A.qperm = pl->d_qperm;
  A.ncols = pl->d_ncols;
  A.ukeys = pl->d_keys;
  A.hc = pl->hc;
  return A;
}

}  // namespace

// Query-layout geometry of a plan (usk.h USK_LAYOUT_QUERY; ledger L32, L34).  Per layer:
//  * every key group of 8 units must have one N (the 8 cells of a slice word are read at one column);
//  * key groups of one class (all of them when the layer's groups share a class) keep their order;
//    with several classes the groups are ordered by (class, group) -- a permutation the class map
//    already fixes, so no index is stored -- and chunks end at class boundaries;
//  * chunk width: 256 units when rows_k * maxN_k * 512 bytes fit shared memory, else 128, else 64
//    (identity layers: one width for the whole layer, from its widest units);
//  * chunk k takes M_k * maxN_k * 2 * CW_k bytes (M_k, maxN_k: the largest rows / N of its units).
usk_status qlayout_geometry(usk_plan* pl) {
  if (pl->M > kPMaxM) return fail(USK_EUNSUPPORTED, "query layout: at most 4 sketch rows");
  pl->h_qc_off.clear();
  pl->h_qc_N.clear();
  pl->h_qc_q0.clear();
  pl->h_qc_n.clear();
  pl->h_qc_M.clear();
  pl->h_qc_cw.clear();
  pl->h_qperm.assign((size_t)(pl->U / kQGroup), 0);
  const int64_t smem_cap = 227 * 1024 - (kPHdr + kPRtab + 1024 + kPZero);  // usk.h: 226,240 B per chunk
  auto M_of = [&](int64_t u) {
    const int c = pl->h_cls[u];
    return c < (int)pl->Mc.size() ? pl->Mc[c] : pl->M;
  };
  int64_t off = 0, chunk = 0;
  for (int l = 0; l < pl->n_layers; ++l) {
    LayerGeom& L = pl->layers[l];
    L.qoff = off;
    L.qchunk0 = chunk;
    L.qruns.clear();
    const int64_t ub = L.unit_begin, G = L.n_units / kQGroup;
    for (int64_t u = 0; u < L.n_units; u += kQGroup)
      for (int v = 1; v < kQGroup; ++v)
        if (pl->h_ncols[ub + u + v] != pl->h_ncols[ub + u])
          return fail(USK_EUNSUPPORTED, "query layout: a key group of layer " + std::to_string(l) +
                                            " mixes column counts (importance classes split the group)");
    // group order: by class of the group's first unit (stable); identity when one class
    std::vector<int32_t> order((size_t)G);
    for (int64_t g = 0; g < G; ++g) order[g] = (int32_t)g;
    bool multi = false;
    for (int64_t g = 1; g < G && !multi; ++g) multi = pl->h_cls[ub + 8 * g] != pl->h_cls[ub];
    if (multi)
      std::stable_sort(order.begin(), order.end(),
                       [&](int32_t a, int32_t b) { return pl->h_cls[ub + 8 * (int64_t)a] < pl->h_cls[ub + 8 * (int64_t)b]; });
    for (int64_t g = 0; g < G; ++g) pl->h_qperm[(size_t)(ub / kQGroup + g)] = order[g];
    L.qperm = multi;
    auto unit_at = [&](int64_t q) { return ub + 8 * (int64_t)order[q >> 3] + (q & 7); };  // query pos -> unit
    auto width_for = [&](int64_t mr, int64_t mx) -> int {
      for (int cw : {256, 128, 64})
        if (mr * mx * 2 * cw <= smem_cap) return cw;
      return 0;
    };
    int fixed_cw = 0;
    if (!multi) {  // one width for the layer
      int mr = 1;
      for (int64_t u = 0; u < L.n_units; ++u) mr = std::max(mr, M_of(ub + u));
      fixed_cw = width_for(mr, L.max_ncols);
      if (!fixed_cw)
        return fail(USK_EUNSUPPORTED, "query layout: a 64-unit chunk of layer " + std::to_string(l) +
                                          " (rows x max N x 128 B) exceeds shared memory");
    }
    int64_t pad = 0;  // padding cells of existing units (N_u < maxN_k or M_u < M_k)
    L.qchunks = 0;
    for (int64_t q = 0; q < L.n_units;) {
      // the chunk's class run ends at the next class boundary (multi) or the layer end
      int64_t run_end = L.n_units;
      if (multi) {
        const uint8_t c0 = pl->h_cls[unit_at(q)];
        run_end = q;
        while (run_end < L.n_units && pl->h_cls[unit_at(run_end)] == c0) run_end += kQGroup;
      }
      int cw = fixed_cw;
      int64_t e = 0;
      int32_t mx = 1, mr = 1;
      if (multi) {  // the widest chunk whose units fit
        cw = 0;
        for (int w : {256, 128, 64}) {
          e = std::min<int64_t>(q + w, run_end);
          mx = 1;
          mr = 1;
          for (int64_t t = q; t < e; ++t) {
            mx = std::max(mx, pl->h_ncols[unit_at(t)]);
            mr = std::max(mr, M_of(unit_at(t)));
          }
          if ((int64_t)mr * mx * 2 * w <= smem_cap) {
            cw = w;
            break;
          }
        }
        if (!cw)
          return fail(USK_EUNSUPPORTED, "query layout: a 64-unit chunk of layer " + std::to_string(l) +
                                            " (rows x max N x 128 B) exceeds shared memory");
      } else {
        e = std::min<int64_t>(q + cw, L.n_units);
        for (int64_t t = q; t < e; ++t) {
          mx = std::max(mx, pl->h_ncols[unit_at(t)]);
          mr = std::max(mr, M_of(unit_at(t)));
        }
      }
      for (int64_t t = q; t < e; ++t) {
        const int64_t u = unit_at(t);
        pad += (int64_t)mr * mx - (pl->h_offsets[u + 1] - pl->h_offsets[u]);
      }
      if (L.qruns.empty() || L.qruns.back().cw != cw) L.qruns.push_back({L.qchunks, 0, cw});
      ++L.qruns.back().n;
      pl->h_qc_off.push_back(off);
      pl->h_qc_N.push_back(mx);
      pl->h_qc_q0.push_back((int32_t)q);
      pl->h_qc_n.push_back((int32_t)(e - q));
      pl->h_qc_M.push_back(mr);
      pl->h_qc_cw.push_back(cw);
      off += (int64_t)mr * mx * 2 * cw;
      ++chunk;
      ++L.qchunks;
      q = e;
    }
    // the kernels take identity layers' chunk starts and rows arithmetically (c * CW, all M rows);
    // a one-class layer with fewer rows than the plan (per-class rows) reads the tables instead
    for (int c = 0; c < L.qchunks && !L.qperm; ++c)
      if (pl->h_qc_M[L.qchunk0 + c] != pl->M) L.qperm = 1;
    L.qcw = L.qruns.empty() ? 256 : L.qruns[0].cw;
    L.qmixed = L.qruns.size() > 1;
    L.qbytes = off - L.qoff;
    // the layout stays (nearly) a bijection of the cells
    const int64_t cells = pl->h_offsets[ub + L.n_units] - pl->h_offsets[ub];
    if (pad * 16 > cells)
      return fail(USK_EUNSUPPORTED, "query layout: chunks would pad layer " + std::to_string(l) + " by " +
                                        std::to_string(pad * 100 / std::max<int64_t>(cells, 1)) +
                                        "% of its cells (units of different N or rows share chunks); use the "
                                        "unit-major layout");
  }
  pl->h_qc_off.push_back(off);
  pl->qtotal = off;
  const size_t nch = pl->h_qc_N.size();
  USK_CUDA(cudaMalloc(&pl->d_qc_off, sizeof(int64_t) * pl->h_qc_off.size()));
  USK_CUDA(cudaMalloc(&pl->d_qc_N, sizeof(int32_t) * std::max<size_t>(nch, 1)));
  USK_CUDA(cudaMalloc(&pl->d_qc_aux, sizeof(int32_t) * 4 * std::max<size_t>(nch, 1)));
  USK_CUDA(cudaMalloc(&pl->d_qperm, sizeof(int32_t) * std::max<size_t>(pl->h_qperm.size(), 1)));
  USK_CUDA(cudaMemcpy(pl->d_qc_off, pl->h_qc_off.data(), sizeof(int64_t) * pl->h_qc_off.size(), cudaMemcpyHostToDevice));
  if (nch) {
    USK_CUDA(cudaMemcpy(pl->d_qc_N, pl->h_qc_N.data(), sizeof(int32_t) * nch, cudaMemcpyHostToDevice));
    USK_CUDA(cudaMemcpy(pl->d_qc_aux, pl->h_qc_q0.data(), sizeof(int32_t) * nch, cudaMemcpyHostToDevice));
    USK_CUDA(cudaMemcpy(pl->d_qc_aux + nch, pl->h_qc_n.data(), sizeof(int32_t) * nch, cudaMemcpyHostToDevice));
    USK_CUDA(cudaMemcpy(pl->d_qc_aux + 2 * nch, pl->h_qc_M.data(), sizeof(int32_t) * nch, cudaMemcpyHostToDevice));
    USK_CUDA(cudaMemcpy(pl->d_qc_aux + 3 * nch, pl->h_qc_cw.data(), sizeof(int32_t) * nch, cudaMemcpyHostToDevice));
  }
  if (!pl->h_qperm.empty())
    USK_CUDA(cudaMemcpy(pl->d_qperm, pl->h_qperm.data(), sizeof(int32_t) * pl->h_qperm.size(), cudaMemcpyHostToDevice));
  // k_qpack's per-chunk layer tables (uploaded once here, not per build call)
  std::vector<int64_t> lay(2 * std::max<size_t>(nch, 1), 0);
  for (int l = 0; l < pl->n_layers; ++l) {
    const LayerGeom& L = pl->layers[l];
    for (int c = 0; c < L.qchunks; ++c) {
      lay[L.qchunk0 + c] = L.unit_begin;
      lay[nch + L.qchunk0 + c] = L.qperm ? L.unit_begin / kQGroup : -1;
    }
  }
  USK_CUDA(cudaMalloc(&pl->d_qc_lay, sizeof(int64_t) * lay.size()));
  USK_CUDA(cudaMemcpy(pl->d_qc_lay, lay.data(), sizeof(int64_t) * lay.size(), cudaMemcpyHostToDevice));
  // the build's fused write-out for table-driven layers: every key group's query position and chunk
  const size_t G = pl->h_qperm.size();
  std::vector<int32_t> qg(2 * std::max<size_t>(G, 1), 0);
  for (int l = 0; l < pl->n_layers; ++l) {
    const LayerGeom& L = pl->layers[l];
    const int64_t gb = L.unit_begin / kQGroup;
    for (int c = 0; c < L.qchunks; ++c) {
      const int64_t a = L.qchunk0 + c;
      for (int32_t q = pl->h_qc_q0[a]; q < pl->h_qc_q0[a] + pl->h_qc_n[a]; q += kQGroup) {
        const int64_t g = gb + pl->h_qperm[gb + q / kQGroup];
        qg[g] = q;
        qg[G + g] = (int32_t)a;
      }
    }
  }
  USK_CUDA(cudaMalloc(&pl->d_qg, sizeof(int32_t) * qg.size()));
  USK_CUDA(cudaMemcpy(pl->d_qg, qg.data(), sizeof(int32_t) * qg.size(), cudaMemcpyHostToDevice));
  return USK_OK;
}

// usk_build on a query-layout plan: the unit-major build (K2) into a stream-ordered scratch buffer,
// then k_qpack writes the requested layers' chunks.
usk_status launch_qbuild(const usk_plan* pl, const void* const* weights, const int32_t* layer_ids, int32_t n,
                         void* sketch, cudaStream_t st) {
  if (n == 0) return USK_OK;
  static const int force_pack = env_int("USK_QBUILD_PACK", 0);
  if (!force_pack && build_qfast_ok(pl, layer_ids, n)) return launch_build_qfast(pl, weights, layer_ids, n, sketch, st);
  void* tmp = nullptr;
  const size_t tmp_bytes = (size_t)pl->total_cells * 2 + 512;
  USK_CUDA(cudaMallocAsync(&tmp, tmp_bytes, st));
  usk_status s = launch_build(pl, weights, layer_ids, n, tmp, st);
  const int64_t nch = (int64_t)pl->h_qc_N.size();
  const int64_t* d_u = pl->d_qc_lay;  // per-chunk layer tables (plan)
  // byte ranges of the requested layers, merged when adjacent
  std::vector<std::pair<int64_t, int64_t>> rg;
  for (int32_t k = 0; k < n; ++k) {
    const LayerGeom& L = pl->layers[layer_ids ? layer_ids[k] : k];
    rg.push_back({L.qoff, L.qoff + L.qbytes});
  }
  std::sort(rg.begin(), rg.end());
  std::vector<std::pair<int64_t, int64_t>> mg;
  for (auto& r : rg) {
    if (!mg.empty() && mg.back().second == r.first) mg.back().second = r.second;
    else mg.push_back(r);
  }
  for (size_t a = 0; s == USK_OK && a < mg.size(); a += 16) {
    PackRanges R{};
    R.n = (int32_t)std::min<size_t>(16, mg.size() - a);
    R.pre[0] = 0;
    for (int r = 0; r < R.n; ++r) {
      R.lo[r] = mg[a + r].first;
      R.hi[r] = mg[a + r].second;
      R.pre[r + 1] = R.pre[r] + (R.hi[r] - R.lo[r]) / 16;
    }
    if (R.pre[R.n] == 0) continue;
    k_qpack<<<(unsigned)((R.pre[R.n] + 255) / 256), 256, 0, st>>>(
        R, reinterpret_cast<const uint16_t*>(tmp), pl->d_qc_off, pl->d_qc_N, d_u, d_u + nch, pl->d_qc_aux,
        pl->d_qperm, pl->d_offsets, pl->d_ncols, pl->d_nrows, nch, reinterpret_cast<uint4*>(sketch));
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) s = cuda_fail(e, "k_qpack");
    else count_launch();
  }
  (void)cudaFreeAsync(tmp, st);
  return s;
}

size_t qgemv_batch_workspace_bytes(const usk_plan* pl, const int32_t* layers, const int64_t* o0, const int64_t* o1,
                                   int n) {
  size_t b = 0;
  for (int k = 0; k < n; ++k) b += layer_ws_bytes(pl->layers[layers[k]].qchunks, o1[k] - o0[k]);
  return b + 256;  // + the split-K control block (two counters, left zero)
}

// entries of one chunk width: every run of that width of the call's layers (ledger L34: a class-ordered
// layer has runs of several widths; the others one run)
struct PEntry {
  int k;  // index in the call
  LayerGeom::QRun run;
};

std::vector<PEntry> entries_of_width(const usk_plan* pl, const int32_t* layers, const std::vector<int>& ks, int cw) {
  std::vector<PEntry> es;
  for (int k : ks)
    for (const auto& r : pl->layers[layers[k]].qruns)
      if (r.cw == cw) es.push_back({k, r});
  return es;
}

void fill_entry(const usk_plan* pl, PLayer& Ly, const LayerGeom& L, const LayerGeom::QRun& r) {
  Ly.unit_base = L.unit_begin;
  Ly.chunk0 = L.qchunk0 + r.c0;
  Ly.n_chunks = r.n;
  Ly.pc0 = r.c0;
  Ly.perm = L.qperm;
  (void)pl;
}

// K4p over entries of one chunk width (partials only)
usk_status qgemv_compute(const usk_plan* pl, const void* sketch, const std::vector<PEntry>& es, int cw,
                         const int32_t* layers, const int64_t* o0, const int64_t* o1, const std::vector<char*>& ws_of,
                         const void* x, int32_t x_dtype, cudaStream_t st) {
  const int64_t in = pl->layers[layers[es[0].k]].in;
  PArgs A = p_base(pl, sketch, in);
  A.x = x;
  bool any_perm = false;
  for (const PEntry& e : es) {
    const LayerGeom& L = pl->layers[layers[e.k]];
    PLayer& Ly = A.layer[A.n_layers++];
    fill_entry(pl, Ly, L, e.run);
    Ly.o_begin = o0[e.k];
    Ly.rows = o1[e.k] - o0[e.k];
    Ly.CP = partial_stride(L.qchunks);
    Ly.partial = reinterpret_cast<float*>(ws_of[e.k]);
    any_perm |= L.qperm != 0;
  }
  static const int xpf = env_int("USK_XPF", 1), forced_sr = env_int("USK_QSR", 0);
  A.x_prefetch = any_perm ? 0 : xpf;
  // subtile height: 16 rows; 8 when a 16-row launch gives each SM fewer than ~9 subtiles for its 16
  // warps (in-graph trace, Llama-3.2-1B o: 1.74 vs 1.99 us; q|k|v at ~10.7 per SM: 2.66 vs 2.57)
  int64_t items16 = 0;
  for (int k = 0; k < A.n_layers; ++k) items16 += (int64_t)A.layer[k].n_chunks * ((A.layer[k].rows + 15) / 16);
  int SR = forced_sr ? forced_sr : (items16 < 9 * (int64_t)device_sm_count() ? 8 : 16);
  const bool tab = any_perm || cw == 64;
  if (tab && SR == 4) SR = 8;
  A.items = 0;
  for (int k = 0; k < A.n_layers; ++k) {
    PLayer& Ly = A.layer[k];
    Ly.n_sub = (int32_t)((Ly.rows + SR - 1) / SR);
    Ly.item_begin = A.items;
    A.items += (int64_t)Ly.n_chunks * Ly.n_sub;
  }
  const void* kern = pick_kernel(true, x_dtype == USK_BF16, pl->M, SR, cw / 32, tab);
  int grid = 0;
  size_t smem = 0;
  usk_status s = p_prepare(pl, A, kern, true, grid, smem, SR, tab);
  if (s != USK_OK) return s;
  A.n_ctas = grid;
  return p_launch(kern, A, grid, kPThreads, smem, st);
}

// the split-K reduction of the call's layers (one launch, after every compute launch of the call)
usk_status qreduce_launch(const usk_plan* pl, const void* sketch, const std::vector<int>& ks, const int32_t* layers,
                          const int64_t* o0, const int64_t* o1, const std::vector<char*>& ws_of, void* const* y,
                          int32_t y_dtype, cudaStream_t st, const usk_peers* peers, int n, unsigned int* done) {
  PArgs A = p_base(pl, sketch, pl->layers[layers[ks[0]]].in);
  A.y_bf16 = y_dtype == USK_BF16;
  int max_chunks = 1;
  for (int k : ks) {
    const LayerGeom& L = pl->layers[layers[k]];
    PLayer& Ly = A.layer[A.n_layers++];
    Ly.unit_base = L.unit_begin;
    Ly.chunk0 = L.qchunk0;
    Ly.o_begin = o0[k];
    Ly.rows = o1[k] - o0[k];
    Ly.row_begin = A.rows;
    Ly.n_chunks = L.qchunks;
    Ly.CP = partial_stride(L.qchunks);
    Ly.y = y[k];
    Ly.partial = reinterpret_cast<float*>(ws_of[k]);
    A.rows += Ly.rows;
    max_chunks = std::max(max_chunks, L.qchunks);
  }
  A.red_lanes = 1;
  while (A.red_lanes < 32 && 4 * A.red_lanes < max_chunks) A.red_lanes *= 2;
  if (peers) {
    A.n_peers = peers->n_peers;
    A.my_rank = peers->my_rank;
    for (int q = 0; q < peers->n_peers; ++q) {
      for (int k = 0; k < (int)ks.size(); ++k) A.ypeer[q][k] = peers->y_peer[(size_t)q * n + ks[k]];
      A.sig[q] = peers->sig_peer[q];
    }
    A.epoch = peers->epoch;
    A.done = done;
  }
  (void)ensure_func_attr((const void*)k_qreduce, (int)cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  const int rgrid = (int)((A.rows * A.red_lanes + kPRedThreads - 1) / kPRedThreads);
  A.timeline = trace_slot(rgrid);
  return p_launch((const void*)k_qreduce, A, rgrid, kPRedThreads, 0, st);
}

usk_status launch_qgemv_batch(const usk_plan* pl, const void* sketch, const int32_t* layers, const int64_t* o0,
                              const int64_t* o1, int n, const void* x, int32_t x_dtype, void* const* y, int32_t y_dtype,
                              void* ws, cudaStream_t st, const usk_peers* peers) {
  // workspace: the layers' partials in call order (qgemv_batch_workspace_bytes).  One K4p launch per
  // chunk width present (256 / 128 / 64 units), then ONE reduce launch over all the call's layers.
  std::vector<char*> ws_of(n);
  char* w = reinterpret_cast<char*>(ws);
  std::vector<int> ks;
  for (int k = 0; k < n; ++k) {
    const LayerGeom& L = pl->layers[layers[k]];
    ws_of[k] = w;
    w += layer_ws_bytes(L.qchunks, o1[k] - o0[k]);
    if (o1[k] > o0[k]) ks.push_back(k);
  }
  if (ks.empty()) return USK_OK;
  unsigned int* done = reinterpret_cast<unsigned int*>(w);  // control block after the partials
  for (int cw : {256, 128, 64}) {
    std::vector<PEntry> es = entries_of_width(pl, layers, ks, cw);
    for (size_t a = 0; a < es.size(); a += kPMaxLayers) {
      std::vector<PEntry> part(es.begin() + a, es.begin() + std::min(es.size(), a + kPMaxLayers));
      usk_status s = qgemv_compute(pl, sketch, part, cw, layers, o0, o1, ws_of, x, x_dtype, st);
      if (s != USK_OK) return s;
    }
  }
  return qreduce_launch(pl, sketch, ks, layers, o0, o1, ws_of, y, y_dtype, st, peers, n, done);
}

usk_status launch_peer_wait(const usk_plan* pl, const usk_peers* peers, cudaStream_t st) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(1);
  cfg.blockDim = dim3(32);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  USK_CUDA(cudaLaunchKernelEx(&cfg, k_peer_wait, (const uint32_t*)peers->sig_peer[peers->my_rank], peers->n_peers,
                              peers->epoch, pl->d_err));
  count_launch();
  return USK_OK;
}

// K3p over several layers (usk_reconstruct, usk_reconstruct_batch): layers sharing in_features, full
// or partial row ranges; one launch per chunk width present, at most kPMaxLayers runs per launch
usk_status qrecon_launch(const usk_plan* pl, const void* sketch, const int32_t* layers, const int64_t* r0,
                         const int64_t* r1, void* const* w_out, const int64_t* ld, int n, cudaStream_t st) {
  const LayerGeom& L0 = pl->layers[layers[0]];
  std::vector<int> ks;
  for (int k = 0; k < n; ++k)
    if (r1[k] > r0[k]) ks.push_back(k);
  for (int cw : {256, 128, 64}) {
    std::vector<PEntry> es = entries_of_width(pl, layers, ks, cw);
    for (size_t a = 0; a < es.size(); a += kPMaxLayers) {
      PArgs A = p_base(pl, sketch, L0.in);
      for (size_t e = a; e < std::min(es.size(), a + kPMaxLayers); ++e) {
        const int k = es[e].k;
        const LayerGeom& L = pl->layers[layers[k]];
        const int64_t rows = r1[k] - r0[k];
        PLayer& Ly = A.layer[A.n_layers++];
        fill_entry(pl, Ly, L, es[e].run);
        Ly.o_begin = r0[k];
        Ly.rows = rows;
        Ly.n_sub = (int32_t)((rows + 15) / 16);
        Ly.w_out = w_out[k];
        Ly.ld_out = ld[k];
        Ly.st_al = (ld[k] % 8 == 0) && (reinterpret_cast<uintptr_t>(w_out[k]) % 16 == 0);
        Ly.item_begin = A.items;
        Ly.row_begin = A.rows;
        A.items += (int64_t)Ly.n_chunks * Ly.n_sub;
        A.rows += rows;
      }
      bool tab = cw == 64;
      for (int k = 0; k < A.n_layers; ++k) tab |= A.layer[k].perm != 0;
      const void* kern = pick_kernel(false, false, pl->M, 16, cw / 32, tab);
      int grid = 0;
      size_t smem = 0;
      usk_status s = p_prepare(pl, A, kern, false, grid, smem, 16, tab);
      if (s == USK_OK) s = p_launch(kern, A, grid, kPThreads, smem, st);
      if (s != USK_OK) return s;
    }
  }
  return USK_OK;
}

usk_status launch_qreconstruct(const usk_plan* pl, const void* sketch, int32_t l, int64_t r0, int64_t r1, void* w_out,
                               int64_t ld, cudaStream_t st) {
  return qrecon_launch(pl, sketch, &l, &r0, &r1, &w_out, &ld, 1, st);
}

usk_status launch_qreconstruct_batch(const usk_plan* pl, const void* sketch, const int32_t* layers, int n,
                                     void* const* w_out, const int64_t* ld, cudaStream_t st) {
  // consecutive runs of layers with one in_features, at most kPMaxLayers per launch
  for (int a = 0; a < n;) {
    int b = a + 1;
    while (b < n && b - a < kPMaxLayers && pl->layers[layers[b]].in == pl->layers[layers[a]].in) ++b;
    std::vector<int64_t> r0(b - a, 0), r1(b - a);
    for (int k = a; k < b; ++k) r1[k - a] = pl->layers[layers[k]].out;
    usk_status s = qrecon_launch(pl, sketch, layers + a, r0.data(), r1.data(), w_out + a, ld + a, b - a, st);
    if (s != USK_OK) return s;
    a = b;
  }
  return USK_OK;
}

}  // namespace usk
