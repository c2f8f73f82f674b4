// plan.cu -- K1: salient-weight-aware sketch space allocation on the device.
//
// PAPER.md:320-334 (§3.4: "assign I_j / sum_i I_i x Mem(Sketch) as the space of sketch state
// for each weight matrix row"; "layer-wise importance is estimated by the mean of row
// importance"), categories PAPER.md:523-528.  Deterministic integer reading: DESIGN.md
// "Allocation".  Pipeline (all on `stream`):
//   k_unit_scores   s_u = sequential fp64 mean of the unit's saliency   (one thread / unit;
//                   USK-XG: of its key group's, ledger L33)
//   k_scope_max     s_max per budget scope (max of non-negative doubles = max of their bits)
//   k_sort_keys     q_u = floor(s_u / s_max * 2^24); key = (scope << 25) | (2^24 - q_u)
//   cub radix sort  stable: rank by (q desc, u asc) inside each scope
//   k_classes       class = floor(rank * C / U_scope); n_c, W_c = sum q_u L_u (u64 atomics, exact)
//   k_geometry      per scope: N_c = max(min_cols, floor(T W_c / (W n_c M_c))) with water-filling
//                   and largest remainder (unsigned __int128)            (one thread / scope)
//                   M_c = the class's sketch rows (usk_params.class_rows, ledger L30; else M)
//   k_unit_sizes    ncols, nrows = M_c, per-unit hash key K_u, size = M_c * N
//   k_scan_*        device-wide exclusive prefix scan of sizes -> unit offsets
#include <cub/device/device_radix_sort.cuh>

#include <cmath>
#include <cstring>

#include "common.cuh"

namespace usk {
namespace {

constexpr int kErrNonFinite = 1;
constexpr int kErrBudget = 2;
constexpr int kErrInval = 4;

constexpr int kMaxClasses = 64;
struct ClassRows {
  int32_t m[kMaxClasses];  // sketch rows per class
};

struct PlanDev {
  const int64_t* unit_base;   // [L+1]
  const int64_t* in_feat;     // [L]
  const int64_t* numel;       // [L]
  const float* const* sal;    // [L] device pointers (may be null entries)
  int32_t L, gran, g, C, M;
  int32_t key_shift;          // USK-XG (ledger L32): unit t takes the key of group t >> 3
};

__device__ __forceinline__ int find_layer(const int64_t* unit_base, int L, int64_t u) {
  int lo = 0, hi = L;  // unit_base[lo] <= u < unit_base[hi]
  while (hi - lo > 1) {
    int mid = (lo + hi) >> 1;
    if (unit_base[mid] <= u) lo = mid; else hi = mid;
  }
  return lo;
}

__global__ void k_unit_scores(PlanDev P, int64_t U, double* s_u, int* err) {
  int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (u >= U) return;
  int l = find_layer(P.unit_base, P.L, u);
  int64_t t = u - P.unit_base[l];
  int64_t j0, j1;
  if (P.gran == USK_GRAN_ROW) {
    // USK-XG (ledger L33): a unit scores by its key group's mean, so a group shares class and N
    const int64_t Ul = P.unit_base[l + 1] - P.unit_base[l];
    const int64_t t0 = (t >> P.key_shift) << P.key_shift;
    const int64_t t1 = min(t0 + ((int64_t)1 << P.key_shift), Ul);
    j0 = t0 * P.g; j1 = t1 * P.g;
  } else { j0 = 0; j1 = P.in_feat[l]; }
  const float* s = P.sal[l];
  double acc = 0.0;
  for (int64_t j = j0; j < j1; ++j) {
    double v = s ? (double)s[j] : 1.0;
    if (!(v >= 0.0) || isinf(v)) { atomicOr(err, kErrInval); v = 0.0; }
    acc += v;
  }
  s_u[u] = acc / (double)(j1 - j0);
}

// warp-aggregated atomics: lanes with equal keys combine first, the group leader does one atomic
__device__ __forceinline__ void group_max_u64(unsigned long long* dst, unsigned key, unsigned long long v) {
  const unsigned mask = __match_any_sync(0xffffffffu, key);
  unsigned long long m = v;
  for (unsigned b = mask; b; b &= b - 1) m = max(m, __shfl_sync(mask, v, __ffs(b) - 1));
  if ((threadIdx.x & 31) == (unsigned)(__ffs(mask) - 1) && dst) atomicMax(dst, m);
}

__device__ __forceinline__ void group_add_u64(unsigned long long* dst, unsigned key, unsigned long long v) {
  const unsigned mask = __match_any_sync(0xffffffffu, key);
  unsigned long long sum = 0;
  for (unsigned b = mask; b; b &= b - 1) sum += __shfl_sync(mask, v, __ffs(b) - 1);
  if ((threadIdx.x & 31) == (unsigned)(__ffs(mask) - 1) && dst) atomicAdd(dst, sum);
}

__global__ void k_scope_max(PlanDev P, int64_t U, const double* s_u, unsigned long long* smax) {
  const int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const bool ok = u < U;
  const int sc = !ok ? -1 : (P.gran != USK_GRAN_LAYER) ? find_layer(P.unit_base, P.L, u) : 0;
  const unsigned long long v = ok ? (unsigned long long)__double_as_longlong(s_u[u]) : 0ull;  // s_u >= 0
  group_max_u64(ok ? &smax[sc] : nullptr, (unsigned)sc, v);
}

__global__ void k_sort_keys(PlanDev P, int64_t U, const double* s_u, const unsigned long long* smax,
                            uint32_t* q, uint64_t* keys, uint32_t* vals) {
  int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (u >= U) return;
  int sc = (P.gran != USK_GRAN_LAYER) ? find_layer(P.unit_base, P.L, u) : 0;
  double mx = __longlong_as_double((long long)smax[sc]);
  uint32_t qu = (mx > 0.0) ? (uint32_t)floor((s_u[u] / mx) * 16777216.0) : 1u;
  q[u] = qu;
  keys[u] = ((uint64_t)sc << 25) | (uint64_t)(16777216u - qu);
  vals[u] = (uint32_t)u;
}

__global__ void k_classes(PlanDev P, int64_t U, const uint64_t* keys_sorted,
                          const uint32_t* vals_sorted, const uint32_t* q, const int64_t* scope_begin,
                          const int64_t* scope_units, uint8_t* cls,
                          unsigned long long* n_c, unsigned long long* W_c) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const bool ok = r < U;
  int64_t slot = -1;
  unsigned long long w = 0;
  if (ok) {
    const int sc = (int)(keys_sorted[r] >> 25);
    const uint32_t u = vals_sorted[r];
    const int64_t rank = r - scope_begin[sc];
    const int c = (int)((rank * (int64_t)P.C) / scope_units[sc]);
    cls[u] = (uint8_t)c;
    const unsigned long long Lu = (P.gran == USK_GRAN_LAYER) ? (unsigned long long)P.numel[u] : 1ull;
    slot = (int64_t)sc * P.C + c;
    w = (unsigned long long)q[u] * Lu;
  }
  // consecutive ranks share (scope, class): aggregate inside the warp before the atomics
  group_add_u64(ok ? &n_c[slot] : nullptr, (unsigned)slot, 1ull);
  group_add_u64(ok ? &W_c[slot] : nullptr, (unsigned)slot, w);
}

// One block (one thread) per scope: proportional share, water-filled floor, largest remainder.
__global__ void k_geometry(int32_t C, ClassRows Mc, int32_t min_cols, const int64_t* T_scope,
                           const unsigned long long* n_c, const unsigned long long* W_c, int32_t* N_c,
                           int* err) {
  typedef unsigned __int128 u128;
  __shared__ u128 num[kMaxClasses], den[kMaxClasses];
  __shared__ int64_t Nv[kMaxClasses];
  __shared__ uint64_t key[kMaxClasses];
  __shared__ bool active[kMaxClasses], done[kMaxClasses];
  if (threadIdx.x != 0) return;
  const int sc = blockIdx.x;
  const unsigned long long* n = n_c + (int64_t)sc * C;
  const unsigned long long* W = W_c + (int64_t)sc * C;
  int32_t* N = N_c + (int64_t)sc * C;
  const int64_t T = T_scope[sc];
  int64_t floor_cells = 0;
  for (int c = 0; c < C; ++c) floor_cells += (int64_t)n[c] * Mc.m[c] * min_cols;
  if (floor_cells > T) {
    atomicOr(err, kErrBudget);
    for (int c = 0; c < C; ++c) N[c] = min_cols;
    return;
  }
  for (int c = 0; c < C; ++c) active[c] = n[c] > 0;
  for (;;) {
    u128 Wa = 0;
    int64_t Ta = T;
    bool changed = false;
    for (int c = 0; c < C; ++c) {
      if (n[c] == 0) continue;
      if (active[c]) Wa += W[c]; else Ta -= (int64_t)n[c] * Mc.m[c] * min_cols;
    }
    for (int c = 0; c < C; ++c) {
      if (!active[c]) continue;
      num[c] = (u128)Ta * W[c];
      den[c] = Wa * (u128)n[c] * (u128)Mc.m[c];
      Nv[c] = den[c] == 0 ? 0 : (int64_t)(num[c] / den[c]);
      if (Nv[c] < min_cols) { active[c] = false; changed = true; }
    }
    if (!changed) break;
  }
  for (int c = 0; c < C; ++c) if (!active[c]) Nv[c] = min_cols;
  int64_t left = T;
  for (int c = 0; c < C; ++c) left -= (int64_t)n[c] * Mc.m[c] * Nv[c];
  // remainder order: (floor(frac * 2^32) desc, c asc), by repeated selection (C <= 64)
  for (int c = 0; c < C; ++c) {
    key[c] = active[c] ? (uint64_t)(((num[c] % den[c]) << 32) / den[c]) : 0;
    done[c] = !active[c];
  }
  for (;;) {
    int best = -1;
    for (int c = 0; c < C; ++c)
      if (!done[c] && (best < 0 || key[c] > key[best])) best = c;
    if (best < 0) break;
    done[best] = true;
    int64_t need = (int64_t)n[best] * Mc.m[best];
    if (need <= left) { Nv[best] += 1; left -= need; }
  }
  for (int c = 0; c < C; ++c) N[c] = (int32_t)Nv[c];
}

__global__ void k_unit_sizes(PlanDev P, ClassRows Mc, int64_t U, uint64_t seed, const uint8_t* cls,
                             const int32_t* N_c, int32_t* ncols, uint8_t* nrows, uint32_t* ukeys,
                             int64_t* sizes) {
  int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (u >= U) return;
  int l = find_layer(P.unit_base, P.L, u);
  int sc = (P.gran != USK_GRAN_LAYER) ? l : 0;
  int64_t t = (P.gran != USK_GRAN_LAYER) ? u - P.unit_base[l] : 0;
  int32_t N = N_c[(int64_t)sc * P.C + cls[u]];
  ncols[u] = N;
  const int32_t m = Mc.m[cls[u]];
  nrows[u] = (uint8_t)m;
  sizes[u] = (int64_t)m * N;
  const uint64_t kt = (uint64_t)t >> P.key_shift;
  ukeys[u] = (uint32_t)splitmix64(seed ^ splitmix64(((uint64_t)(uint32_t)l << 32) | kt));
}

// ---- device-wide exclusive scan of int64 sizes -> offsets[0..U] (3 kernels) ----
constexpr int kScanThreads = 1024;
constexpr int kScanItems = 4;
constexpr int kScanTile = kScanThreads * kScanItems;

__device__ int64_t block_exclusive_scan(int64_t v, int64_t* sh, int64_t* total) {
  // warp scan then scan of warp sums
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int64_t x = v;
  for (int o = 1; o < 32; o <<= 1) {
    int64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sh[w] = x;
  __syncthreads();
  if (w == 0) {
    int64_t s = (lane < (int)(blockDim.x >> 5)) ? sh[lane] : 0;
    for (int o = 1; o < 32; o <<= 1) {
      int64_t y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    sh[32 + lane] = s;
  }
  __syncthreads();
  int64_t warp_prefix = (w == 0) ? 0 : sh[32 + w - 1];
  *total = sh[32 + (blockDim.x >> 5) - 1];
  __syncthreads();
  return warp_prefix + x - v;
}

__global__ void k_scan_tiles(const int64_t* in, int64_t U, int64_t* tile_sums) {
  __shared__ int64_t sh[64];
  int64_t base = blockIdx.x * (int64_t)kScanTile + threadIdx.x * kScanItems;
  int64_t s = 0;
  for (int k = 0; k < kScanItems; ++k) s += (base + k < U) ? in[base + k] : 0;
  int64_t total;
  block_exclusive_scan(s, sh, &total);
  if (threadIdx.x == 0) tile_sums[blockIdx.x] = total;
}

__global__ void k_scan_sums(int64_t* tile_sums, int64_t n_tiles) {
  __shared__ int64_t sh[64];
  int64_t carry = 0;
  for (int64_t b = 0; b < n_tiles; b += blockDim.x) {
    int64_t i = b + threadIdx.x;
    int64_t v = i < n_tiles ? tile_sums[i] : 0;
    int64_t total;
    int64_t ex = block_exclusive_scan(v, sh, &total);
    if (i < n_tiles) tile_sums[i] = carry + ex;
    carry += total;
  }
}

__global__ void k_scan_apply(const int64_t* in, int64_t U, const int64_t* tile_prefix, int64_t* out) {
  __shared__ int64_t sh[64];
  int64_t base = blockIdx.x * (int64_t)kScanTile + threadIdx.x * kScanItems;
  int64_t v[kScanItems];
  int64_t s = 0;
  for (int k = 0; k < kScanItems; ++k) { v[k] = (base + k < U) ? in[base + k] : 0; s += v[k]; }
  int64_t total;
  int64_t ex = block_exclusive_scan(s, sh, &total) + tile_prefix[blockIdx.x];
  for (int k = 0; k < kScanItems; ++k) {
    if (base + k < U) out[base + k] = ex;
    ex += v[k];
  }
}

__global__ void k_scan_last(const int64_t* in, int64_t U, int64_t* out) {
  out[U] = out[U - 1] + in[U - 1];
}

// position mixes of the g = 1 layouts for the build's bulk copies: per output row o,
// {R_0, R_1, R_2} mod 2^23 and 0 (16 B, so a stage of rows is one contiguous copy)
__global__ void k_R4_table(HashConsts hc, int64_t n, uint4* R4) {
  const int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (o >= n) return;
  const uint32_t p = (uint32_t)o;
  R4[o] = make_uint4(fmix32(p ^ hc.rho[0]) & 0x7FFFFFu, fmix32(p ^ hc.rho[1]) & 0x7FFFFFu,
                     fmix32(p ^ hc.rho[2]) & 0x7FFFFFu, 0u);
}

inline unsigned blocks_for(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

template <class T>
cudaError_t dmalloc(T** p, size_t count, cudaStream_t st) {
  return cudaMallocAsync((void**)p, sizeof(T) * (count ? count : 1), st);
}

}  // namespace

usk_status build_plan_device(usk_plan* pl, const float* const* saliency, cudaStream_t st) {
  const int32_t L = pl->n_layers;
  const int64_t U = pl->U;
  const int32_t C = pl->C;
  const int32_t n_scopes = (pl->gran != USK_GRAN_LAYER) ? L : 1;

  std::vector<int64_t> h_unit_base(L + 1), h_in(L), h_numel(L), h_T(n_scopes), h_sbegin(n_scopes),
      h_sunits(n_scopes);
  for (int l = 0; l < L; ++l) {
    h_unit_base[l] = pl->layers[l].unit_begin;
    h_in[l] = pl->layers[l].in;
    h_numel[l] = pl->layers[l].out * pl->layers[l].in;
  }
  h_unit_base[L] = U;
  for (int s = 0; s < n_scopes; ++s) {
    if (pl->gran != USK_GRAN_LAYER) {
      h_T[s] = pl->layers[s].cells_T;
      h_sbegin[s] = pl->layers[s].unit_begin;
      h_sunits[s] = pl->layers[s].n_units;
    } else {
      h_T[s] = pl->layers[0].cells_T;
      h_sbegin[s] = 0;
      h_sunits[s] = U;
    }
  }
  std::vector<const float*> h_sal(L, nullptr);
  if (saliency)
    for (int l = 0; l < L; ++l) h_sal[l] = saliency[l];

  // temporaries
  int64_t *d_unit_base, *d_in, *d_numel, *d_T, *d_sbegin, *d_sunits, *d_sizes, *d_tiles;
  const float** d_sal;
  double* d_s;
  unsigned long long *d_smax, *d_nc, *d_Wc;
  uint32_t *d_q, *d_vals, *d_vals2;
  uint64_t *d_keys, *d_keys2;
  int32_t* d_Nc;
  const int64_t n_tiles = (U + kScanTile - 1) / kScanTile;
  USK_CUDA(dmalloc(&d_unit_base, L + 1, st));
  USK_CUDA(dmalloc(&d_in, L, st));
  USK_CUDA(dmalloc(&d_numel, L, st));
  USK_CUDA(dmalloc(&d_T, n_scopes, st));
  USK_CUDA(dmalloc(&d_sbegin, n_scopes, st));
  USK_CUDA(dmalloc(&d_sunits, n_scopes, st));
  USK_CUDA(dmalloc(&d_sal, L, st));
  USK_CUDA(dmalloc(&d_s, U, st));
  USK_CUDA(dmalloc(&d_smax, n_scopes, st));
  USK_CUDA(dmalloc(&d_nc, (size_t)n_scopes * C, st));
  USK_CUDA(dmalloc(&d_Wc, (size_t)n_scopes * C, st));
  USK_CUDA(dmalloc(&d_q, U, st));
  USK_CUDA(dmalloc(&d_vals, U, st));
  USK_CUDA(dmalloc(&d_vals2, U, st));
  USK_CUDA(dmalloc(&d_keys, U, st));
  USK_CUDA(dmalloc(&d_keys2, U, st));
  USK_CUDA(dmalloc(&d_Nc, (size_t)n_scopes * C, st));
  USK_CUDA(dmalloc(&d_sizes, U, st));
  USK_CUDA(dmalloc(&d_tiles, n_tiles, st));
  USK_CUDA(cudaMemcpyAsync(d_unit_base, h_unit_base.data(), sizeof(int64_t) * (L + 1), cudaMemcpyHostToDevice, st));
  USK_CUDA(cudaMemcpyAsync(d_in, h_in.data(), sizeof(int64_t) * L, cudaMemcpyHostToDevice, st));
  USK_CUDA(cudaMemcpyAsync(d_numel, h_numel.data(), sizeof(int64_t) * L, cudaMemcpyHostToDevice, st));
  USK_CUDA(cudaMemcpyAsync(d_T, h_T.data(), sizeof(int64_t) * n_scopes, cudaMemcpyHostToDevice, st));
  USK_CUDA(cudaMemcpyAsync(d_sbegin, h_sbegin.data(), sizeof(int64_t) * n_scopes, cudaMemcpyHostToDevice, st));
  USK_CUDA(cudaMemcpyAsync(d_sunits, h_sunits.data(), sizeof(int64_t) * n_scopes, cudaMemcpyHostToDevice, st));
  USK_CUDA(cudaMemcpyAsync(d_sal, h_sal.data(), sizeof(float*) * L, cudaMemcpyHostToDevice, st));
  USK_CUDA(cudaMemsetAsync(d_smax, 0, sizeof(unsigned long long) * n_scopes, st));
  USK_CUDA(cudaMemsetAsync(d_nc, 0, sizeof(unsigned long long) * n_scopes * C, st));
  USK_CUDA(cudaMemsetAsync(d_Wc, 0, sizeof(unsigned long long) * n_scopes * C, st));
  USK_CUDA(cudaMemsetAsync(pl->d_err, 0, sizeof(int), st));

  PlanDev P{d_unit_base, d_in, d_numel, d_sal, L, pl->gran, pl->g, C, pl->M, pl->hash_api == USK_HASH_XG ? 3 : 0};
  const int T256 = 256;
  k_unit_scores<<<blocks_for(U, T256), T256, 0, st>>>(P, U, d_s, pl->d_err);
  USK_LAUNCHED("k_unit_scores");
  k_scope_max<<<blocks_for(U, T256), T256, 0, st>>>(P, U, d_s, d_smax);
  USK_LAUNCHED("k_scope_max");
  k_sort_keys<<<blocks_for(U, T256), T256, 0, st>>>(P, U, d_s, d_smax, d_q, d_keys, d_vals);
  USK_LAUNCHED("k_sort_keys");
  int end_bit = 25;
  while ((1ll << (end_bit - 25)) < n_scopes) ++end_bit;
  size_t temp_bytes = 0;
  USK_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, temp_bytes, d_keys, d_keys2, d_vals, d_vals2, (int)U, 0,
                                           end_bit, st));
  void* d_temp;
  USK_CUDA(cudaMallocAsync(&d_temp, temp_bytes, st));
  USK_CUDA(cub::DeviceRadixSort::SortPairs(d_temp, temp_bytes, d_keys, d_keys2, d_vals, d_vals2, (int)U, 0,
                                           end_bit, st));
  count_launch();
  k_classes<<<blocks_for(U, T256), T256, 0, st>>>(P, U, d_keys2, d_vals2, d_q, d_sbegin, d_sunits, pl->d_cls,
                                                  d_nc, d_Wc);
  USK_LAUNCHED("k_classes");
  ClassRows Mc{};
  for (int c = 0; c < C && c < kMaxClasses; ++c) Mc.m[c] = pl->Mc[c];
  k_geometry<<<(unsigned)n_scopes, 32, 0, st>>>(C, Mc, pl->min_cols, d_T, d_nc, d_Wc, d_Nc,
                                                      pl->d_err);
  USK_LAUNCHED("k_geometry");
  k_unit_sizes<<<blocks_for(U, T256), T256, 0, st>>>(P, Mc, U, pl->seed, pl->d_cls, d_Nc, pl->d_ncols, pl->d_nrows,
                                                     pl->d_keys, d_sizes);
  USK_LAUNCHED("k_unit_sizes");
  k_scan_tiles<<<(unsigned)n_tiles, kScanThreads, 0, st>>>(d_sizes, U, d_tiles);
  USK_LAUNCHED("k_scan_tiles");
  k_scan_sums<<<1, kScanThreads, 0, st>>>(d_tiles, n_tiles);
  USK_LAUNCHED("k_scan_sums");
  k_scan_apply<<<(unsigned)n_tiles, kScanThreads, 0, st>>>(d_sizes, U, d_tiles, pl->d_offsets);
  USK_LAUNCHED("k_scan_apply");
  k_scan_last<<<1, 1, 0, st>>>(d_sizes, U, pl->d_offsets);
  USK_LAUNCHED("k_scan_last");
  k_R4_table<<<blocks_for(pl->max_pos, T256), T256, 0, st>>>(pl->hc, pl->max_pos, pl->d_R4);
  USK_LAUNCHED("k_R4_table");

  int h_err = 0;
  pl->h_ncols.resize(U);
  pl->h_offsets.resize(U + 1);
  pl->h_cls.resize(U);
  USK_CUDA(cudaMemcpyAsync(&h_err, pl->d_err, sizeof(int), cudaMemcpyDeviceToHost, st));
  USK_CUDA(cudaMemcpyAsync(pl->h_ncols.data(), pl->d_ncols, sizeof(int32_t) * U, cudaMemcpyDeviceToHost, st));
  USK_CUDA(cudaMemcpyAsync(pl->h_offsets.data(), pl->d_offsets, sizeof(int64_t) * (U + 1), cudaMemcpyDeviceToHost, st));
  USK_CUDA(cudaMemcpyAsync(pl->h_cls.data(), pl->d_cls, U, cudaMemcpyDeviceToHost, st));
  void* frees[] = {d_unit_base, d_in, d_numel, d_T, d_sbegin, d_sunits, (void*)d_sal, d_s, d_smax, d_nc, d_Wc,
                   d_q, d_vals, d_vals2, d_keys, d_keys2, d_Nc, d_sizes, d_tiles, d_temp};
  for (void* p : frees) USK_CUDA(cudaFreeAsync(p, st));
  USK_CUDA(cudaStreamSynchronize(st));
  USK_CUDA(cudaMemsetAsync(pl->d_err, 0, sizeof(int), st));
  if (h_err & kErrInval) return fail(USK_EINVAL, "saliency must be finite and >= 0");
  if (h_err & kErrBudget) return fail(USK_EBUDGET, "infeasible floor: sum_c n_c * M * min_cols > T");
  (void)kErrNonFinite;
  return USK_OK;
}

}  // namespace usk
