// query.cu -- K3 reconstruct, K4 sketch-GEMV (decode), K6 importance.
//
// Query of one weight (Eq. 3 + Eq. 5; §3.1 "hash ... retrieved by the above
// indices in a batch ... interpreting these intermediate results"):
//   w'(o, j) = the bonded cell of maximum |.| over rows i < M (ties -> non-negative, L1/L2).
//
// Fast path (ROW granularity, one input dimension per unit).  Work is cut into ITEMS =
// (layer, chunk of TJ = 32*UPL consecutive units, block of 32*warps output rows), ordered
// layer-major, chunk-major.  A persistent grid (<= resident CTAs) takes contiguous item ranges,
// so a CTA stages a chunk's cells once and reuses them over many row blocks.  Lane L owns units
// UPL*L+v; their cells are staged into shared memory as rho codes
//     rho = rotl(bits_hi, 1) ^ 1 = (mag << 1) | (1 - sign)
// at byte address  cells + 4*(v*32*maxMN + k*32 + L)  -- always bank L, so the M random
// gathers of a warp never conflict.  The Eq. 5 select is an integer max (VIMNMX3 for M=3) and
// rotr(rho, 1) is the IEEE pattern of -w', so the GEMV multiplies by -x (exact).
// Per weight and lane: 1 LOP3 (R(o) ^ K_u) + M x (IMAD, IMAD.HI, LEA, LDS) + max + SHF + FFMA.
// Missing units of a ragged chunk point at a shared "zero" cell (rho of +0) with x = 0, so the
// inner loop has no branches.
//
// GEMV: a warp computes 32 rows; lane L then holds its units' share of 32 row sums, which a
// padded shared-memory transpose turns into one row per lane.  Split-K partials are reduced in
// a fixed chunk order by whichever CTA completes a row block last (deterministic, no float
// atomics).  Programmatic dependent launch: the first chunk is staged (sketch only) before
// griddepcontrol.wait, so it overlaps the previous kernel.  usk_linear_batch puts several
// linears that share x (q|k|v, gate|up) in one launch.
#include <algorithm>

#include "common.cuh"

namespace usk {
namespace {

constexpr int kQThreads = 512;
constexpr int kQWarps = kQThreads / 32;
constexpr int kRB = kQWarps * 32;                 // rows per item
constexpr int kMaxBatch = 8;
constexpr int kScratchWords = kQWarps * 32 * 33;  // GEMV transpose scratch

__device__ __forceinline__ uint32_t lds32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}

struct QLayer {
  int64_t unit_base;   // global unit id of the layer's first unit
  int64_t o_begin;     // first output row
  int64_t rows;        // rows in [o_begin, o_end)
  int32_t n_chunks;    // unit chunks of TJ
  int32_t n_rb;        // row blocks of kRB
  int32_t item_begin;  // first item of this layer in the launch
  int32_t pad;
  // gemv
  void* y;
  float* partial;      // [n_chunks][rows]
  uint32_t* counters;  // [n_rb]
  // reconstruct
  void* w_out;
  int64_t ld_out;
};

struct QArgs {
  QLayer layer[kMaxBatch];
  int32_t n_layers;
  int32_t total_items;
  int32_t M;
  int32_t maxMN;       // smem slot stride (cells) = max over the launch's layers
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
};

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
  const int lane = threadIdx.x & 31;
  const E* sk = reinterpret_cast<const E*>(A.sketch);
  {
    const int ul = threadIdx.x % TJ;
    if (ul < nu) {
      const int64_t u = Ly.unit_base + j0 + ul;
      const int64_t off = A.offsets[u];
      const int mn = A.M * A.ncols[u];
      const int L = ul / UPL, v = ul % UPL;
      uint32_t* dst = cells + v * 32 * A.maxMN + L;
#pragma unroll 8
      for (int k = threadIdx.x / TJ; k < mn; k += kQThreads / TJ) {
        uint32_t b = (uint32_t)sk[off + k];
        if (sizeof(E) == 2) b <<= 16;
        dst[k * 32] = rotl1(b) ^ 1u;
      }
    }
  }
  const uint32_t cbase = smem_u32(cells), zbase = smem_u32(zero);
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

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// ------------------------------------------------------------------ K3 / K4 persistent kernel
template <typename E, int UPL, int MT, int HASH, bool GEMV>
__global__ void __launch_bounds__(kQThreads) k_query_fast(const __grid_constant__ QArgs A) {
  constexpr int TJ = 32 * UPL;
  extern __shared__ __align__(16) uint32_t qsm[];
  __shared__ int s_last;
  float* scratch = reinterpret_cast<float*>(qsm);                // GEMV only
  uint32_t* Rs = qsm + (GEMV ? kScratchWords : 0);
  uint32_t* zero = Rs + kRB;
  uint32_t* cells = zero + 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

  const int it0 = (int)(((int64_t)blockIdx.x * A.total_items) / gridDim.x);
  const int it1 = (int)(((int64_t)(blockIdx.x + 1) * A.total_items) / gridDim.x);
  int cur_li = -1, cur_chunk = -1;
  bool waited = false;
  LaneState<UPL, MT> S;
  float nx[UPL];
#pragma unroll
  for (int v = 0; v < UPL; ++v) nx[v] = 0.f;

  for (int it = it0; it < it1; ++it) {
    int li = 0;
    while (li + 1 < A.n_layers && A.layer[li + 1].item_begin <= it) ++li;
    const QLayer& Ly = A.layer[li];
    const int local = it - Ly.item_begin;
    const int chunk = local / Ly.n_rb, rbk = local % Ly.n_rb;
    const int64_t j0 = (int64_t)chunk * TJ;
    const int nu = (int)min((int64_t)TJ, A.in - j0);
    const int64_t r0 = (int64_t)rbk * kRB;
    const int rows = (int)min((int64_t)kRB, Ly.rows - r0);

    if constexpr (GEMV) {
      if (it == it1 - 1 && waited) pdl_trigger();  // let the next kernel's prologue start
    }
    __syncthreads();  // previous item is done with cells / Rs
    if (li != cur_li || chunk != cur_chunk) {
      stage_chunk<E, UPL, MT>(A, Ly, j0, nu, cells, zero, S);
      cur_li = li;
      cur_chunk = chunk;
      if constexpr (GEMV) {
        if (!waited) {  // x may be written by the previous kernel on the stream
          pdl_wait();
          waited = true;
        }
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
    }
    {
      const int r = threadIdx.x;  // kQThreads == kRB
      Rs[r] = A.R[Ly.o_begin + r0 + min(r, rows - 1)];
      if (threadIdx.x < 32) zero[threadIdx.x] = 1u;  // rho(+0)
    }
    __syncthreads();

    const int s0 = warp * 32;
    if constexpr (GEMV) {
      float acc[32];
#pragma unroll
      for (int r = 0; r < 32; ++r) {
        const uint32_t Rv = Rs[s0 + r];
        float a = 0.f;
#pragma unroll
        for (int v = 0; v < UPL; ++v)
          a = fmaf(nx[v], __uint_as_float(rotr1(select_rho<UPL, MT, HASH>(A, S, v, Rv, Ly.o_begin + r0 + s0 + r))), a);
        acc[r] = a;
      }
      // transpose through padded shared memory: lane r sums row r over the 32 lanes (fixed order)
      float* sc = scratch + warp * (32 * 33);
#pragma unroll
      for (int r = 0; r < 32; ++r) sc[r * 33 + lane] = acc[r];
      __syncwarp();
      float s = 0.f;
#pragma unroll
      for (int k = 0; k < 32; ++k) s += sc[lane * 33 + k];
      if (s0 + lane < rows) Ly.partial[(int64_t)chunk * Ly.rows + r0 + s0 + lane] = s;
      // ---- deterministic split-K: the CTA completing row block rbk sums its chunks in order
      __threadfence();
      __syncthreads();
      if (threadIdx.x == 0) s_last = (atomicAdd(&Ly.counters[rbk], 1u) == (uint32_t)Ly.n_chunks - 1);
      __syncthreads();
      if (s_last) {
        __threadfence();
        const int r = threadIdx.x;
        if (r < rows) {
          float t = 0.f;
          const float* p = Ly.partial + r0 + r;
          for (int c = 0; c < Ly.n_chunks; ++c) t += __ldcg(p + (int64_t)c * Ly.rows);
          if (A.y_bf16) {
            const uint32_t bb = __float_as_uint(t);
            reinterpret_cast<uint16_t*>(Ly.y)[r0 + r] = (uint16_t)((bb + 0x7FFFu + ((bb >> 16) & 1u)) >> 16);
          } else {
            reinterpret_cast<float*>(Ly.y)[r0 + r] = t;
          }
        }
        if (threadIdx.x == 0) Ly.counters[rbk] = 0u;  // leave the workspace zeroed
      }
    } else {
      const bool full_tile = (nu == TJ);
#pragma unroll 4
      for (int r = 0; r < 32; ++r) {
        if (s0 + r >= rows) break;
        const int64_t o = Ly.o_begin + r0 + s0 + r;
        const uint32_t Rv = Rs[s0 + r];
        uint32_t wb[UPL];
#pragma unroll
        for (int v = 0; v < UPL; ++v) wb[v] = rotr1(select_rho<UPL, MT, HASH>(A, S, v, Rv, o)) ^ 0x80000000u;
        E* dst = reinterpret_cast<E*>(Ly.w_out) + (r0 + s0 + r) * Ly.ld_out + j0 + UPL * lane;
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
  }
  if constexpr (GEMV) {
    if (!waited) pdl_wait();
    pdl_trigger();
  }
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

struct Geom {
  int upl = 0;
  int maxMN = 0;
  size_t smem = 0;
  int items = 0;
  int grid = 0;
  std::vector<int> n_chunks, n_rb;
};

size_t smem_bytes(bool gemv, int upl, int maxMN) {
  return (gemv ? (size_t)kScratchWords * 4 : 0) + (size_t)kRB * 4 + 128 + (size_t)32 * upl * maxMN * 4;
}

constexpr size_t kSmemMax = 220 * 1024;
constexpr size_t kSmemPerSM = 228 * 1024;

// Pick units-per-lane and the persistent grid for a launch covering `layers` (rows each).
// Larger UPL amortises the per-row work (R(o) load, transpose) over more weights; it must still
// leave >= 148 items so every SM gets work.
Geom geometry(const usk_plan* pl, const int32_t* layers, const int64_t* rows, int n, bool gemv) {
  Geom G;
  for (int k = 0; k < n; ++k) G.maxMN = std::max(G.maxMN, pl->M * pl->layers[layers[k]].max_ncols);
  const int64_t in = pl->layers[layers[0]].in;
  auto items_for = [&](int upl) {
    int it = 0;
    for (int k = 0; k < n; ++k)
      it += (int)((in + 32 * upl - 1) / (32 * upl)) * (int)((rows[k] + kRB - 1) / kRB);
    return it;
  };
  int best = 0;
  for (int upl : {4, 2, 1}) {
    if (smem_bytes(gemv, upl, G.maxMN) > kSmemMax) continue;
    best = upl;
    if (items_for(upl) >= 148) break;
  }
  if (!best) return G;
  G.upl = best;
  G.smem = smem_bytes(gemv, best, G.maxMN);
  for (int k = 0; k < n; ++k) {
    G.n_chunks.push_back((int)((in + 32 * best - 1) / (32 * best)));
    G.n_rb.push_back((int)((rows[k] + kRB - 1) / kRB));
    G.items += G.n_chunks.back() * G.n_rb.back();
  }
  const int per_sm = std::max<int>(1, std::min<int>(4, (int)(kSmemPerSM / (G.smem + 1024))));
  const int resident = 148 * std::min(per_sm, 2048 / kQThreads);
  G.grid = std::min(G.items, resident);
  return G;
}

size_t layer_ws_bytes(int n_chunks, int n_rb, int64_t rows) {
  const size_t p = ((size_t)n_chunks * rows * 4 + 255) / 256 * 256;
  return p + ((size_t)n_rb * 4 + 255) / 256 * 256;
}

QArgs base_args(const usk_plan* pl, const void* sketch, int64_t in, const Geom& G) {
  QArgs A{};
  A.M = pl->M;
  A.maxMN = G.maxMN;
  A.total_items = G.items;
  A.in = in;
  A.sketch = sketch;
  A.ncols = pl->d_ncols;
  A.offsets = pl->d_offsets;
  A.ukeys = pl->d_keys;
  A.R = pl->d_R;
  A.hc = pl->hc;
  return A;
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

usk_status launch_q(void* kern, const QArgs& A, int grid, size_t smem, bool pdl, cudaStream_t st) {
  // max dynamic smem is raised once per kernel (callers warm up before any graph capture)
  static std::vector<void*> raised;
  if (std::find(raised.begin(), raised.end(), kern) == raised.end()) {
    USK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemMax));
    raised.push_back(kern);
  }
  int occ = 1;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kQThreads, smem) != cudaSuccess || occ < 1) occ = 1;
  int sms = 148;
  {
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  grid = std::min(grid, sms * occ);  // persistent: every CTA resident
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
  void* args[] = {const_cast<QArgs*>(&A)};
  USK_CUDA(cudaLaunchKernelExC(&cfg, kern, args));
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
  std::vector<int64_t> rows(n);
  for (int k = 0; k < n; ++k) rows[k] = o1[k] - o0[k];
  Geom G = geometry(pl, layers, rows.data(), n, true);
  if (!G.upl) return 256;
  size_t b = 0;
  for (int k = 0; k < n; ++k) b += layer_ws_bytes(G.n_chunks[k], G.n_rb[k], rows[k]);
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
    int item = 0;
    for (int k = 0; k < n; ++k) {
      const size_t wsb = layer_ws_bytes(G.n_chunks[k], G.n_rb[k], rows[k]);
      if (rows[k] == 0) {
        w += wsb;
        continue;
      }
      QLayer& Ly = A.layer[A.n_layers++];
      Ly.unit_base = pl->layers[layers[k]].unit_begin;
      Ly.o_begin = o0[k];
      Ly.rows = rows[k];
      Ly.n_chunks = G.n_chunks[k];
      Ly.n_rb = G.n_rb[k];
      Ly.item_begin = item;
      item += Ly.n_chunks * Ly.n_rb;
      Ly.y = y[k];
      Ly.partial = reinterpret_cast<float*>(w);
      const size_t p = ((size_t)Ly.n_chunks * rows[k] * 4 + 255) / 256 * 256;
      Ly.counters = reinterpret_cast<uint32_t*>(w + p);
      w += wsb;
    }
    if (!A.n_layers) return USK_OK;
    A.total_items = item;
    void* k = pick_fast(G.upl, true, pl->dtype == USK_BF16, pl->M, pl->hash);
    return launch_q(k, A, std::min(G.grid, item), G.smem, true, st);
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
    Ly.n_rb = G.n_rb[0];
    Ly.item_begin = 0;
    Ly.w_out = w_out;
    Ly.ld_out = ld;
    void* k = pick_fast(G.upl, false, pl->dtype == USK_BF16, pl->M, pl->hash);
    return launch_q(k, A, G.grid, G.smem, false, st);
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
