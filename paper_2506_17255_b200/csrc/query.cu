// query.cu -- K3 reconstruct, K4 sketch-GEMV (decode), K6 importance.
//
// Query of one weight (Eq. 3 + Eq. 5; §3.1 "hash ... retrieved by the above
// indices in a batch ... interpreting these intermediate results"):
//   w'(o, j) = the bonded cell of maximum |.| over rows i < M (ties -> non-negative, L1/L2).
// Shared-memory layout (fast path, ROW, one input dim per unit): a CTA owns TJ = 32*UPL
// consecutive units; lane L owns units UPL*L+v, whose cells sit at word
// (v*32*maxMN + k*32 + L) -- always bank L -- as rho codes  rho = rotl(bits_hi, 1) ^ 1
// = (mag << 1) | (1 - sign).  The select is then an integer max and rotr(rho, 1) is the
// bit pattern of -w', so the GEMV multiplies by -x (exact: only the sign bit moves).
// Lanes therefore run over units (input dims) and warps over output rows; the per-row
// position mix R(o) is staged once per CTA.  Split-K partial sums are reduced in a fixed
// order by the last CTA of each row block (deterministic, no float atomics).
#include <algorithm>

#include "common.cuh"

namespace usk {
namespace {

constexpr int kQThreads = 256;
constexpr int kQWarps = kQThreads / 32;

struct QueryArgs {
  const void* sketch;
  const int32_t* ncols;
  const int64_t* offsets;
  const uint32_t* ukeys;
  const uint32_t* R;
  HashConsts hc;
  int64_t unit_base;  // global unit id of the layer's first unit
  int64_t in;
  int64_t o_begin, o_end;
  int32_t M, maxMN;
  int32_t rb_rows;    // rows per CTA (row block)
  int32_t n_chunks;
  // reconstruct
  void* w_out;
  int64_t ld_out;
  // gemv
  const void* x;
  int32_t x_bf16;
  void* y;
  int32_t y_bf16;
  float* partial;     // [n_chunks][rows]
  uint32_t* counters; // [n_rb]
};

// Stage the CTA's units into shared memory (rho layout) and R(o) for its rows.
template <typename E, int UPL>
__device__ __forceinline__ void stage_units(const QueryArgs& A, int64_t j0, int nu, int64_t r0, int rows,
                                            uint32_t* cells, uint32_t* Rs) {
  constexpr int TJ = 32 * UPL;
  const int stride_v = 32 * A.maxMN;
  const E* sk = reinterpret_cast<const E*>(A.sketch);
  const int ul = threadIdx.x % TJ;
  if (ul < nu) {
    const int64_t u = A.unit_base + j0 + ul;
    const int64_t off = A.offsets[u];
    const int mn = A.M * A.ncols[u];
    const int L = ul / UPL, v = ul % UPL;
    for (int k = threadIdx.x / TJ; k < mn; k += kQThreads / TJ) {
      uint32_t b = (uint32_t)sk[off + k];
      if (sizeof(E) == 2) b <<= 16;
      cells[v * stride_v + k * 32 + L] = rotl1(b) ^ 1u;
    }
  }
  for (int r = threadIdx.x; r < rows; r += kQThreads) Rs[r] = A.R[A.o_begin + r0 + r];
}

template <int UPL, int MR>
struct LaneUnits {
  uint32_t K[UPL], N[UPL];
  int rb[UPL][MR];
  bool valid[UPL];
};

template <int UPL, int MR>
__device__ __forceinline__ void load_lane_units(const QueryArgs& A, int64_t j0, int nu, LaneUnits<UPL, MR>& U) {
  const int lane = threadIdx.x & 31;
  const int stride_v = 32 * A.maxMN;
#pragma unroll
  for (int v = 0; v < UPL; ++v) {
    const int ul = UPL * lane + v;
    U.valid[v] = ul < nu;
    const int64_t u = A.unit_base + j0 + (U.valid[v] ? ul : 0);
    U.K[v] = A.ukeys[u];
    U.N[v] = (uint32_t)A.ncols[u];
#pragma unroll
    for (int i = 0; i < MR; ++i) U.rb[v][i] = v * stride_v + i * (int)U.N[v] * 32 + lane;
  }
}

// rho code of w'(o, unit v of this lane)
template <int UPL, int MT, int HASH, int MR>
__device__ __forceinline__ uint32_t select_rho(const QueryArgs& A, const uint32_t* cells,
                                               const LaneUnits<UPL, MR>& U, int v, uint32_t Rv, int64_t o) {
  const uint32_t h = Rv ^ U.K[v];
  uint32_t best = 0;
#pragma unroll
  for (int i = 0; i < MR; ++i) {
    if (MT == 0 && i >= A.M) break;
    uint32_t idx;
    if constexpr (HASH == USK_HASH_X) idx = __umulhi(h * A.hc.a[i], U.N[v]);
    else idx = (uint32_t)(o % U.N[v]);
    best = max(best, cells[U.rb[v][i] + idx * 32]);
  }
  return best;
}

// ------------------------------------------------------------------ K3: reconstruct
template <typename E, int UPL, int MT, int HASH>
__global__ void __launch_bounds__(kQThreads) k_reconstruct_fast(const __grid_constant__ QueryArgs A) {
  constexpr int TJ = 32 * UPL;
  constexpr int MR = MT > 0 ? MT : 8;
  extern __shared__ __align__(16) uint32_t qsm[];
  uint32_t* Rs = qsm;
  uint32_t* cells = qsm + A.rb_rows;
  const int chunk = blockIdx.x % A.n_chunks;
  const int rbk = blockIdx.x / A.n_chunks;
  const int64_t j0 = (int64_t)chunk * TJ;
  const int nu = (int)min((int64_t)TJ, A.in - j0);
  const int64_t rows_total = A.o_end - A.o_begin;
  const int64_t r0 = (int64_t)rbk * A.rb_rows;
  const int rows = (int)min((int64_t)A.rb_rows, rows_total - r0);
  stage_units<E, UPL>(A, j0, nu, r0, rows, cells, Rs);
  LaneUnits<UPL, MR> U;
  load_lane_units<UPL, MR>(A, j0, nu, U);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  E* out = reinterpret_cast<E*>(A.w_out);
  for (int r = warp; r < rows; r += kQWarps) {
    const int64_t o = A.o_begin + r0 + r;
    const uint32_t Rv = Rs[r];
    uint32_t wb[UPL];
#pragma unroll
    for (int v = 0; v < UPL; ++v) wb[v] = rotr1(select_rho<UPL, MT, HASH, MR>(A, cells, U, v, Rv, o)) ^ 0x80000000u;
    E* dst = out + (r0 + r) * A.ld_out + j0 + UPL * lane;
    if constexpr (sizeof(E) == 2 && UPL == 2) {
      if (U.valid[1]) *reinterpret_cast<uint32_t*>(dst) = __byte_perm(wb[0], wb[1], 0x7632);
      else if (U.valid[0]) dst[0] = (E)(wb[0] >> 16);
    } else if constexpr (sizeof(E) == 2) {
      if (U.valid[0]) dst[0] = (E)(wb[0] >> 16);
    } else {
#pragma unroll
      for (int v = 0; v < UPL; ++v)
        if (U.valid[v]) dst[v] = wb[v];
    }
  }
}

// ------------------------------------------------------------------ K4: sketch-GEMV
// y[o] = sum_j x[j] w'(o, j), o in [o_begin, o_end).  Warp: 32-row subtiles; lane: UPL units.
// After a subtile each lane holds acc[r] (its units' contribution to row r); a transpose
// butterfly leaves the warp's 32 row partials one per lane.
__device__ __forceinline__ void transpose_reduce32(float (&acc)[32], int lane) {
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) {
    const bool up = (lane & m) != 0;
#pragma unroll
    for (int i = 0; i < m; ++i) {
      const float send = up ? acc[i] : acc[i + m];
      const float keep = up ? acc[i + m] : acc[i];
      acc[i] = keep + __shfl_xor_sync(0xffffffffu, send, m);
    }
  }
  // lane now holds, in acc[0], the sum for row r = lane (bit-reversal free: rows were split
  // by their high bits first, so the surviving index is the lane's own row)
}

template <typename E, int UPL, int MT, int HASH>
__global__ void __launch_bounds__(kQThreads) k_gemv_fast(const __grid_constant__ QueryArgs A) {
  constexpr int TJ = 32 * UPL;
  constexpr int MR = MT > 0 ? MT : 8;
  extern __shared__ __align__(16) uint32_t qsm[];
  __shared__ bool s_last;
  uint32_t* Rs = qsm;
  uint32_t* cells = qsm + A.rb_rows;
  const int chunk = blockIdx.x % A.n_chunks;
  const int rbk = blockIdx.x / A.n_chunks;
  const int64_t j0 = (int64_t)chunk * TJ;
  const int nu = (int)min((int64_t)TJ, A.in - j0);
  const int64_t rows_total = A.o_end - A.o_begin;
  const int64_t r0 = (int64_t)rbk * A.rb_rows;
  const int rows = (int)min((int64_t)A.rb_rows, rows_total - r0);
  stage_units<E, UPL>(A, j0, nu, r0, rows, cells, Rs);
  LaneUnits<UPL, MR> U;
  load_lane_units<UPL, MR>(A, j0, nu, U);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float nx[UPL];
#pragma unroll
  for (int v = 0; v < UPL; ++v) {
    const int64_t j = j0 + UPL * lane + v;
    float xv = 0.f;
    if (U.valid[v]) {
      if (A.x_bf16) xv = __uint_as_float((uint32_t)reinterpret_cast<const uint16_t*>(A.x)[j] << 16);
      else xv = reinterpret_cast<const float*>(A.x)[j];
    }
    nx[v] = -xv;  // rotr(rho) decodes to -w'
  }
  __syncthreads();
  float* P = A.partial + (int64_t)chunk * rows_total + r0;
  for (int s0 = warp * 32; s0 < rows; s0 += kQWarps * 32) {
    float acc[32];
#pragma unroll
    for (int r = 0; r < 32; ++r) {
      const int rr = min(s0 + r, rows - 1);
      const uint32_t Rv = Rs[rr];
      const int64_t o = A.o_begin + r0 + rr;
      float a = 0.f;
#pragma unroll
      for (int v = 0; v < UPL; ++v) {
        if (!U.valid[v]) continue;  // ragged unit tile: slot not staged
        const uint32_t best = select_rho<UPL, MT, HASH, MR>(A, cells, U, v, Rv, o);
        a = fmaf(nx[v], __uint_as_float(rotr1(best)), a);
      }
      acc[r] = a;
    }
    transpose_reduce32(acc, lane);
    if (s0 + lane < rows) P[s0 + lane] = acc[0];
  }
  // ---- deterministic split-K: the last CTA of this row block sums chunks in order
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t prev = atomicAdd(&A.counters[rbk], 1u);
    s_last = (prev == (uint32_t)A.n_chunks - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  for (int r = threadIdx.x; r < rows; r += kQThreads) {
    float s = 0.f;
    const float* p = A.partial + r0 + r;
    for (int c = 0; c < A.n_chunks; ++c) s += __ldcg(p + (int64_t)c * rows_total);
    if (A.y_bf16) {
      const uint32_t b = __float_as_uint(s);
      const uint32_t rnd = b + 0x7FFFu + ((b >> 16) & 1u);  // RNE (finite)
      reinterpret_cast<uint16_t*>(A.y)[r0 + r] = (uint16_t)(rnd >> 16);
    } else {
      reinterpret_cast<float*>(A.y)[r0 + r] = s;
    }
  }
  if (threadIdx.x == 0) A.counters[rbk] = 0u;  // leave the workspace zeroed for the next call
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

// ------------------------------------------------------------------ host helpers
int query_upl(const usk_plan* pl, int32_t l, size_t* smem_out, int rb_rows) {
  const LayerGeom& L = pl->layers[l];
  if (pl->gran != USK_GRAN_ROW || pl->g != 1) return 0;
  const int64_t mn = (int64_t)pl->M * L.max_ncols;
  for (int upl = 2; upl >= 1; --upl) {
    const size_t smem = (size_t)rb_rows * 4 + (size_t)32 * upl * mn * 4;
    if (smem <= (upl == 2 ? 100 * 1024 : 200 * 1024)) {
      if (smem_out) *smem_out = smem;
      return upl;
    }
  }
  return 0;
}

struct Geometry {
  int upl = 0;
  int n_chunks = 0, n_rb = 0, rb_rows = 0;
  size_t smem = 0;
};

Geometry gemv_geometry(const usk_plan* pl, int32_t l, int64_t rows) {
  Geometry G;
  const LayerGeom& L = pl->layers[l];
  // first pass at a 1024-row block to pick UPL, then size row blocks for ~3 CTAs per SM
  G.upl = query_upl(pl, l, nullptr, 1024);
  if (!G.upl) return G;
  const int TJ = 32 * G.upl;
  G.n_chunks = (int)((L.in + TJ - 1) / TJ);
  const int64_t target = 148 * 3;
  int64_t n_rb = std::max<int64_t>(1, (target + G.n_chunks - 1) / G.n_chunks);
  int64_t rb = (rows + n_rb - 1) / n_rb;
  rb = std::max<int64_t>(32, ((rb + 31) / 32) * 32);
  rb = std::min<int64_t>(rb, 1024);
  G.rb_rows = (int)rb;
  G.n_rb = (int)((rows + rb - 1) / rb);
  G.upl = query_upl(pl, l, &G.smem, G.rb_rows);
  return G;
}

QueryArgs make_args(const usk_plan* pl, int32_t l, const void* sketch, int64_t o0, int64_t o1) {
  const LayerGeom& L = pl->layers[l];
  QueryArgs A{};
  A.sketch = sketch;
  A.ncols = pl->d_ncols;
  A.offsets = pl->d_offsets;
  A.ukeys = pl->d_keys;
  A.R = pl->d_R;
  A.hc = pl->hc;
  A.unit_base = L.unit_begin;
  A.in = L.in;
  A.o_begin = o0;
  A.o_end = o1;
  A.M = pl->M;
  A.maxMN = pl->M * L.max_ncols;
  return A;
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

#define USK_PICK(KNAME)                                                                          \
  template <typename E, int UPL>                                                                 \
  void* pick_##KNAME(int M, int hash) {                                                          \
    if (hash == USK_HASH_IDENTITY) return (void*)KNAME<E, UPL, 0, USK_HASH_IDENTITY>;            \
    switch (M) {                                                                                 \
      case 1: return (void*)KNAME<E, UPL, 1, USK_HASH_X>;                                        \
      case 2: return (void*)KNAME<E, UPL, 2, USK_HASH_X>;                                        \
      case 3: return (void*)KNAME<E, UPL, 3, USK_HASH_X>;                                        \
      default: return (void*)KNAME<E, UPL, 0, USK_HASH_X>;                                       \
    }                                                                                            \
  }
USK_PICK(k_reconstruct_fast)
USK_PICK(k_gemv_fast)

template <int UPL>
void* pick_fast(bool gemv, bool bf16, int M, int hash) {
  if (gemv) return bf16 ? pick_k_gemv_fast<uint16_t, UPL>(M, hash) : pick_k_gemv_fast<uint32_t, UPL>(M, hash);
  return bf16 ? pick_k_reconstruct_fast<uint16_t, UPL>(M, hash) : pick_k_reconstruct_fast<uint32_t, UPL>(M, hash);
}

usk_status launch_fast_query(void* kern, const QueryArgs& A, unsigned grid, size_t smem, cudaStream_t st) {
  USK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  void* args[] = {const_cast<QueryArgs*>(&A)};
  USK_CUDA(cudaLaunchKernel(kern, dim3(grid), dim3(kQThreads), args, smem, st));
  count_launch();
  return USK_OK;
}

}  // namespace

size_t gemv_workspace_bytes(const usk_plan* pl, int32_t l, int64_t o0, int64_t o1) {
  const int64_t rows = o1 - o0;
  Geometry G = gemv_geometry(pl, l, rows);
  if (!G.upl) return 0;
  const size_t p = (size_t)G.n_chunks * rows * 4;
  return ((p + 255) / 256) * 256 + (size_t)G.n_rb * 4;
}

usk_status launch_reconstruct(const usk_plan* pl, const void* sketch, int32_t l, int64_t r0, int64_t r1, void* w_out,
                              int64_t ld, cudaStream_t st) {
  const LayerGeom& L = pl->layers[l];
  const int64_t rows = r1 - r0;
  if (rows == 0) return USK_OK;
  size_t smem = 0;
  const int rb_rows = 256;
  const int upl = query_upl(pl, l, &smem, rb_rows);
  const bool aligned = ((ld * pl->cell_bytes()) % 4 == 0) && (reinterpret_cast<uintptr_t>(w_out) % 4 == 0);
  if (upl && aligned) {
    QueryArgs A = make_args(pl, l, sketch, r0, r1);
    A.rb_rows = rb_rows;
    A.n_chunks = (int)((L.in + 32 * upl - 1) / (32 * upl));
    A.w_out = w_out;
    A.ld_out = ld;
    const int n_rb = (int)((rows + rb_rows - 1) / rb_rows);
    void* k = upl == 2 ? pick_fast<2>(false, pl->dtype == USK_BF16, pl->M, pl->hash)
                       : pick_fast<1>(false, pl->dtype == USK_BF16, pl->M, pl->hash);
    return launch_fast_query(k, A, (unsigned)(A.n_chunks * n_rb), smem, st);
  }
  GenQ Q = make_genq(pl, l, sketch);
  const int64_t n = rows * L.in;
  k_reconstruct_gen<<<(unsigned)std::min<int64_t>((n + 255) / 256, 148 * 16), 256, 0, st>>>(Q, r0, r1, w_out, ld);
  USK_LAUNCHED("k_reconstruct_gen");
  return USK_OK;
}

usk_status launch_gemv(const usk_plan* pl, const void* sketch, int32_t l, const void* x, int32_t x_dtype, void* y,
                       int32_t y_dtype, int64_t o0, int64_t o1, void* ws, size_t ws_bytes, cudaStream_t st) {
  const int64_t rows = o1 - o0;
  if (rows == 0) return USK_OK;
  Geometry G = gemv_geometry(pl, l, rows);
  if (G.upl) {
    QueryArgs A = make_args(pl, l, sketch, o0, o1);
    A.rb_rows = G.rb_rows;
    A.n_chunks = G.n_chunks;
    A.x = x;
    A.x_bf16 = x_dtype == USK_BF16;
    A.y = y;
    A.y_bf16 = y_dtype == USK_BF16;
    const size_t p = (size_t)G.n_chunks * rows * 4;
    A.partial = reinterpret_cast<float*>(ws);
    A.counters = reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(ws) + ((p + 255) / 256) * 256);
    (void)ws_bytes;
    void* k = G.upl == 2 ? pick_fast<2>(true, pl->dtype == USK_BF16, pl->M, pl->hash)
                         : pick_fast<1>(true, pl->dtype == USK_BF16, pl->M, pl->hash);
    return launch_fast_query(k, A, (unsigned)(G.n_chunks * G.n_rb), G.smem, st);
  }
  GenQ Q = make_genq(pl, l, sketch);
  const int rows_per_block = 8;
  k_gemv_gen<<<(unsigned)((rows + rows_per_block - 1) / rows_per_block), 32 * rows_per_block, 0, st>>>(
      Q, o0, o1, x, x_dtype == USK_BF16, y, y_dtype == USK_BF16);
  USK_LAUNCHED("k_gemv_gen");
  return USK_OK;
}

usk_status launch_importance(const void* A, int32_t a_dtype, int64_t N, int64_t d, float* I, cudaStream_t st) {
  k_importance<<<(unsigned)((d + 255) / 256), 256, 0, st>>>(A, a_dtype == USK_BF16, N, d, I);
  USK_LAUNCHED("k_importance");
  return USK_OK;
}

}  // namespace usk
