// api.cu -- the C ABI (include/usk.h): validation, plan lifetime, dispatch.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <new>
#include <string>
#include <tuple>

#include "common.cuh"

namespace usk {

static thread_local std::string g_last_error;
static thread_local int64_t g_launches = 0;

void set_error(const std::string& msg) { g_last_error = msg; }
usk_status fail(usk_status st, const std::string& msg) {
  g_last_error = msg;
  return st;
}
usk_status cuda_fail(cudaError_t e, const char* what) {
  g_last_error = std::string(what) + ": " + cudaGetErrorString(e);
  (void)cudaGetLastError();  // do not let a non-sticky error leak into the next launch check
  return USK_ECUDA;
}
void count_launch(int n) { g_launches += n; }

// Function attributes apply to the CURRENT device's context: cache them per (device, kernel,
// value), under a lock (concurrent calls on several streams and devices are allowed, usk.h).
static std::mutex g_attr_mu;
cudaError_t ensure_func_attr(const void* kern, int attr, int value) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(g_attr_mu);
  static std::map<std::tuple<int, const void*, int, int>, cudaError_t> done;
  const auto key = std::make_tuple(dev, kern, attr, value);
  auto it = done.find(key);
  if (it != done.end()) return it->second;
  e = cudaFuncSetAttribute(kern, (cudaFuncAttribute)attr, value);
  if (e != cudaSuccess) (void)cudaGetLastError();
  done[key] = e;
  return e;
}
int device_sm_count() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  std::lock_guard<std::mutex> lock(g_attr_mu);
  static std::map<int, int> sms;
  auto it = sms.find(dev);
  if (it != sms.end()) return it->second;
  int n = 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) {
    (void)cudaGetLastError();
    n = 148;
  }
  sms[dev] = n;
  return n;
}

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

static int ceil_log2(int c) {
  int b = 0;
  while ((1 << b) < c) ++b;
  return b;
}

// First level of the two-level allocation (L28): cells per layer from the layer
// importance, exact integer arithmetic (u128); false when the floors exceed T.
static bool layer_cells(int L, const double* imp, const std::vector<int64_t>& numel, const std::vector<int64_t>& Ul,
                        int M, int min_cols, int64_t T, std::vector<int64_t>& Tl) {
  typedef unsigned __int128 u128;
  double smax = 0.0;
  for (int l = 0; l < L; ++l) smax = std::max(smax, imp[l]);
  std::vector<u128> w(L), num(L, 0), den(L, 0);
  std::vector<int> active(L, 1);
  std::vector<int64_t> fl(L);
  int64_t floor_sum = 0;
  for (int l = 0; l < L; ++l) {
    const uint64_t q = smax > 0.0 ? (uint64_t)std::floor((imp[l] / smax) * 16777216.0) : 1u;
    w[l] = (u128)q * (u128)numel[l];
    fl[l] = Ul[l] * M * (int64_t)min_cols;
    floor_sum += fl[l];
  }
  if (floor_sum > T) return false;
  Tl.assign(L, 0);
  for (bool changed = true; changed;) {
    changed = false;
    u128 Wa = 0;
    int64_t Ta = T;
    for (int l = 0; l < L; ++l) {
      if (active[l]) Wa += w[l];
      else Ta -= fl[l];
    }
    for (int l = 0; l < L; ++l) {
      if (!active[l]) continue;
      num[l] = (u128)Ta * w[l];
      den[l] = Wa;
      Tl[l] = Wa == 0 ? 0 : (int64_t)(num[l] / den[l]);
      if (Tl[l] < fl[l]) active[l] = 0, changed = true;
    }
  }
  int64_t left = T;
  std::vector<std::pair<uint64_t, int>> rem;
  for (int l = 0; l < L; ++l) {
    if (!active[l]) Tl[l] = fl[l];
    left -= Tl[l];
    if (active[l] && den[l] != 0) rem.push_back({(uint64_t)(((num[l] % den[l]) << 32) / den[l]), l});
  }
  std::sort(rem.begin(), rem.end(), [](const std::pair<uint64_t, int>& a, const std::pair<uint64_t, int>& b) {
    return a.first != b.first ? a.first > b.first : a.second < b.second;
  });
  for (size_t k = 0; k < rem.size() && left > 0; ++k, --left) Tl[rem[k].second] += 1;
  return true;
}

static void free_plan(usk_plan* p) {
  if (!p) return;
  void* ptrs[] = {p->d_cls, p->d_ncols, p->d_nrows, p->d_offsets, p->d_keys, p->d_R4, p->d_err, p->d_qc_off, p->d_qc_N, p->d_qc_aux, p->d_qperm, p->d_qc_lay, p->d_qg};
  for (void* q : ptrs)
    if (q) cudaFree(q);
  delete p;
}

}  // namespace usk

using namespace usk;

extern "C" {

const char* usk_status_string(usk_status s) {
  switch (s) {
    case USK_OK: return "USK_OK";
    case USK_EINVAL: return "USK_EINVAL";
    case USK_ESHAPE: return "USK_ESHAPE";
    case USK_EBUDGET: return "USK_EBUDGET";
    case USK_ENONFINITE: return "USK_ENONFINITE";
    case USK_ECUDA: return "USK_ECUDA";
    case USK_EUNSUPPORTED: return "USK_EUNSUPPORTED";
    case USK_ERANGE: return "USK_ERANGE";
  }
  return "USK_UNKNOWN";
}

const char* usk_last_error(void) { return g_last_error.c_str(); }

int64_t usk_launch_count(int32_t reset) {
  int64_t v = g_launches;
  if (reset) g_launches = 0;
  return v;
}

usk_status usk_importance(const void* A, int32_t a_dtype, int64_t N, int64_t d, float* I_out, usk_stream stream) {
  if (!A || !I_out) return fail(USK_EINVAL, "usk_importance: null pointer");
  if (a_dtype != USK_F32 && a_dtype != USK_BF16) return fail(USK_EINVAL, "usk_importance: dtype");
  if (N < 1 || d < 1) return fail(USK_ESHAPE, "usk_importance: N and d must be >= 1");
  return launch_importance(A, a_dtype, N, d, I_out, (cudaStream_t)stream);
}

usk_status usk_plan_allocation(const usk_shape* layers, int32_t n_layers, const float* const* saliency,
                               const usk_params* params, usk_plan** plan_out, usk_stream stream) {
  if (!plan_out) return fail(USK_EINVAL, "usk_plan_allocation: plan_out is null");
  *plan_out = nullptr;
  if (!layers || !params) return fail(USK_EINVAL, "usk_plan_allocation: null layers/params");
  if (n_layers < 1) return fail(USK_ESHAPE, "usk_plan_allocation: n_layers < 1");
  const usk_params& P = *params;
  if (!(P.bpw > 0.0) || !std::isfinite(P.bpw)) return fail(USK_EINVAL, "bpw must be finite and > 0");
  if (P.rows < 1 || P.rows > 8) return fail(USK_EINVAL, "rows must be in [1, 8]");
  if (P.granularity != USK_GRAN_ROW && P.granularity != USK_GRAN_LAYER && P.granularity != USK_GRAN_OUTROW)
    return fail(USK_EINVAL, "granularity");
  if (P.granularity == USK_GRAN_OUTROW && (P.n_classes > 1 || P.dims_per_unit != 1))
    return fail(USK_EINVAL, "OUTROW units form one class (n_classes 0 or 1) with dims_per_unit 1");
  if (P.hash != USK_HASH_X && P.hash != USK_HASH_IDENTITY && P.hash != USK_HASH_XG) return fail(USK_EINVAL, "hash");
  if (P.layout != USK_LAYOUT_UNIT_MAJOR && P.layout != USK_LAYOUT_QUERY) return fail(USK_EINVAL, "layout");
  if (P.layout == USK_LAYOUT_QUERY) {  // usk.h: the query layout's conditions (L32, §4)
    if (P.hash != USK_HASH_XG) return fail(USK_EUNSUPPORTED, "query layout: needs USK_HASH_XG (key groups of 8 units)");
    if (P.granularity != USK_GRAN_ROW || P.dims_per_unit != 1)
      return fail(USK_EUNSUPPORTED, "query layout: ROW units with dims_per_unit 1 only");
    if (P.dtype != USK_BF16 || P.state_bits || P.variant != USK_ABSMAXMIN || P.topk)
      return fail(USK_EUNSUPPORTED, "query layout: raw bf16 states, AbsMaxMin, no Top-K");
    for (int l = 0; l < n_layers; ++l)
      if (layers[l].in_features % 8 != 0) return fail(USK_EUNSUPPORTED, "query layout: in_features % 8 != 0");
  }
  if (P.dtype != USK_F32 && P.dtype != USK_BF16) return fail(USK_EINVAL, "dtype");
  if (P.min_cols < 1) return fail(USK_EINVAL, "min_cols must be >= 1");
  if (P.n_classes < 0 || P.n_classes > 64) return fail(USK_EINVAL, "n_classes must be in [0, 64]");
  if (P.state_bits != 0 && P.state_bits != 4 && P.state_bits != 8) return fail(USK_EINVAL, "state_bits must be 0, 4 or 8");
  const int32_t qG = P.group_size ? P.group_size : 128;
  if (P.variant < USK_ABSMAXMIN || P.variant > USK_COUNTMIN) return fail(USK_EINVAL, "variant");
  if (P.topk < 0) return fail(USK_EINVAL, "topk must be >= 0");
  if (P.topk > 0 && (P.granularity != USK_GRAN_ROW || P.state_bits || P.variant != USK_ABSMAXMIN))
    return fail(USK_EINVAL, "topk: ROW granularity, raw states and AbsMaxMin only");
  if (P.layer_importance) {
    if (P.granularity == USK_GRAN_LAYER || P.state_bits)
      return fail(USK_EINVAL, "layer_importance: ROW granularity with raw states only");
    for (int l = 0; l < n_layers; ++l)
      if (!(P.layer_importance[l] >= 0.0) || !std::isfinite(P.layer_importance[l]))
        return fail(USK_EINVAL, "layer_importance must be finite and >= 0");
  }
  if (P.variant != USK_ABSMAXMIN && P.state_bits) return fail(USK_EUNSUPPORTED, "variants use raw states");
  const int32_t n_cls = P.n_classes > 0 ? P.n_classes : (saliency && P.granularity != USK_GRAN_OUTROW ? 4 : 1);
  int32_t max_rows = P.rows;
  if (P.class_rows) {  // per-class sketch rows (ledger L30)
    if (P.layer_importance) return fail(USK_EINVAL, "class_rows: not with layer_importance");
    if (P.variant != USK_ABSMAXMIN) return fail(USK_EINVAL, "class_rows: AbsMaxMin only");
    max_rows = 0;
    for (int c = 0; c < n_cls; ++c) {
      if (P.class_rows[c] < 1 || P.class_rows[c] > 8) return fail(USK_EINVAL, "class_rows must be in [1, 8]");
      max_rows = std::max(max_rows, P.class_rows[c]);
    }
  }
  if (P.state_bits && (qG < 32 || (qG & (qG - 1)) != 0))
    return fail(USK_EINVAL, "group_size must be a power of two >= 32");
  const int g = P.granularity == USK_GRAN_ROW ? P.dims_per_unit : 1;
  if (P.granularity == USK_GRAN_ROW && g < 1) return fail(USK_EINVAL, "dims_per_unit must be >= 1");
  for (int l = 0; l < n_layers; ++l) {
    if (layers[l].out_features < 1 || layers[l].in_features < 1)
      return fail(USK_ESHAPE, "layer " + std::to_string(l) + " has a zero dimension");
    if (layers[l].out_features * layers[l].in_features > 0xFFFFFFFFll)
      return fail(USK_ESHAPE, "layer " + std::to_string(l) + " exceeds 2^32 weights (32-bit positions)");
    if (P.granularity == USK_GRAN_ROW && layers[l].in_features % g != 0)
      return fail(USK_EINVAL, "dims_per_unit does not divide in_features of layer " + std::to_string(l));
  }
  usk_plan* pl = new (std::nothrow) usk_plan();
  if (!pl) return fail(USK_ECUDA, "out of host memory");
  pl->n_layers = n_layers;
  pl->M = max_rows;
  pl->Mc.assign(n_cls, P.rows);
  if (P.class_rows) pl->Mc.assign(P.class_rows, P.class_rows + n_cls);
  pl->gran = P.granularity;
  pl->g = g;
  pl->C = n_cls;
  pl->min_cols = P.min_cols;
  pl->hash = P.hash == USK_HASH_XG ? USK_HASH_X : P.hash;  // same kernels; grouped keys in d_keys
  pl->hash_api = P.hash;
  pl->layout = P.layout;
  pl->variant = P.variant;
  pl->topk = P.topk;
  pl->dtype = P.dtype;
  pl->bpw = P.bpw;
  pl->seed = P.seed;
  pl->q = P.state_bits;
  pl->G = P.state_bits ? qG : 128;
  const int state_bits = P.dtype == USK_BF16 ? 16 : 32;
  for (int i = 0; i < 8; ++i) {  // per-row salts
    pl->hc.rho[i] = (uint32_t)splitmix64(P.seed + 0x200ull + (uint64_t)i);
    pl->hc.kap[i] = (uint32_t)splitmix64(P.seed + 0x300ull + (uint64_t)i);
  }
  cudaGetDevice(&pl->device);

  pl->layers.resize(n_layers);
  int64_t U = 0, numel_all = 0;
  for (int l = 0; l < n_layers; ++l) {
    LayerGeom& L = pl->layers[l];
    L = LayerGeom{};
    L.out = layers[l].out_features;
    L.in = layers[l].in_features;
    L.unit_begin = U;
    L.n_units = P.granularity == USK_GRAN_ROW ? L.in / g : P.granularity == USK_GRAN_OUTROW ? L.out : 1;
    L.scope = P.granularity != USK_GRAN_LAYER ? l : 0;
    U += L.n_units;
    numel_all += L.out * L.in;
    pl->max_out = std::max<int64_t>(pl->max_out, L.out);
    pl->max_pos = std::max<int64_t>(pl->max_pos, std::max(L.out, L.in));
  }
  pl->U = U;
  pl->numel = numel_all;
  std::vector<int64_t> two_T;
  if (P.layer_importance) {  // two-level: one model budget split over the layers first (L28)
    std::vector<int64_t> numel(n_layers), Ul(n_layers);
    int64_t meta_sum = 0;
    for (int l = 0; l < n_layers; ++l) {
      numel[l] = pl->layers[l].out * pl->layers[l].in;
      Ul[l] = pl->layers[l].n_units;
      meta_sum += pl->C > 1 ? Ul[l] * ceil_log2(pl->C) : 0;
    }
    const int64_t budget = (int64_t)std::floor(P.bpw * (double)numel_all);
    if (budget < meta_sum || !layer_cells(n_layers, P.layer_importance, numel, Ul, pl->M, pl->min_cols,
                                          (budget - meta_sum) / state_bits, two_T)) {
      free_plan(pl);
      return fail(USK_EBUDGET, "two-level allocation: the layer floors exceed the model budget");
    }
  }
  if (P.granularity != USK_GRAN_LAYER) {
    for (int l = 0; l < n_layers; ++l) {
      LayerGeom& L = pl->layers[l];
      const int64_t meta = pl->C > 1 ? L.n_units * ceil_log2(pl->C) : 0;
      const int64_t budget =
          P.layer_importance ? two_T[l] * state_bits + meta : (int64_t)std::floor(P.bpw * (double)(L.out * L.in));
      if (budget < meta) {
        free_plan(pl);
        return fail(USK_EBUDGET, "budget smaller than the class map of layer " + std::to_string(l));
      }
      L.budget_bits = budget;
      L.meta_bits = meta;
      // Top-K outliers: (int32 index, state) pairs charged to the layer (L29)
      L.n_out = std::min<int64_t>(pl->topk, L.out * L.in);
      const int64_t side = L.n_out * (32 + state_bits);
      if (budget < meta + side) {
        free_plan(pl);
        return fail(USK_EBUDGET, "Top-K side table exceeds the budget of layer " + std::to_string(l));
      }
      // quantised: ceil(cells/G) groups of q*G code bits + one fp32 scale (layers G-aligned)
      L.cells_T = pl->q ? ((budget - meta - side) / ((int64_t)pl->q * pl->G + 32)) * pl->G
                        : (budget - meta - side) / state_bits;
      pl->budget_bits += budget;
    }
    if (P.layer_importance) pl->budget_bits = (int64_t)std::floor(P.bpw * (double)numel_all);  // one model scope
  } else {
    const int64_t budget = (int64_t)std::floor(P.bpw * (double)numel_all);
    pl->layers[0].budget_bits = budget;
    // quantised: one partial group per layer is reserved (each layer starts a new group)
    pl->layers[0].cells_T =
        pl->q ? std::max<int64_t>(0, budget / ((int64_t)pl->q * pl->G + 32) - n_layers) * pl->G : budget / state_bits;
    pl->budget_bits = budget;
  }
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e = cudaSuccess;
  e = e ? e : cudaMalloc(&pl->d_cls, (size_t)U);
  e = e ? e : cudaMalloc(&pl->d_ncols, sizeof(int32_t) * U);
  e = e ? e : cudaMalloc(&pl->d_nrows, (size_t)U);
  e = e ? e : cudaMalloc(&pl->d_offsets, sizeof(int64_t) * (U + 1));
  e = e ? e : cudaMalloc(&pl->d_keys, sizeof(uint32_t) * U);
  e = e ? e : cudaMalloc(&pl->d_R4, sizeof(uint4) * (pl->max_pos + 32));
  e = e ? e : cudaMalloc(&pl->d_err, sizeof(int));
  if (e != cudaSuccess) {
    free_plan(pl);
    return cuda_fail(e, "usk_plan_allocation: cudaMalloc");
  }
  usk_status s = build_plan_device(pl, saliency, st);
  if (s != USK_OK) {
    cudaStreamSynchronize(st);
    free_plan(pl);
    return s;
  }
  if (pl->q) {
    // each layer's cells start at a multiple of G (groups never straddle layers, so
    // layer-sharded builds quantise independently): shift the prefix-scan offsets on the host
    int64_t shift = 0;
    for (int l = 0; l < n_layers; ++l) {
      const int64_t u0 = pl->layers[l].unit_begin, u1 = u0 + pl->layers[l].n_units;
      const int64_t start = pl->h_offsets[u0] + shift;
      shift += (start + pl->G - 1) / pl->G * pl->G - start;
      for (int64_t u = u0; u < u1; ++u) pl->h_offsets[u] += shift;
    }
    pl->h_offsets[U] += shift;
    e = cudaMemcpy(pl->d_offsets, pl->h_offsets.data(), sizeof(int64_t) * (U + 1), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
      free_plan(pl);
      return cuda_fail(e, "usk_plan_allocation: offsets upload");
    }
  }
  pl->total_cells = pl->q ? (pl->h_offsets[U] + pl->G - 1) / pl->G * pl->G : pl->h_offsets[U];
  if (pl->q) {
    pl->n_groups = pl->total_cells / pl->G;
    pl->scales_off = (pl->code_bytes() + 255) / 256 * 256;
  }
  if (pl->topk) {  // side tables after the cells, layer by layer (16-B aligned pieces)
    int64_t off = (pl->total_cells * pl->cell_bytes() + 255) / 256 * 256;
    for (int l = 0; l < n_layers; ++l) {
      LayerGeom& L = pl->layers[l];
      L.out_off = off;
      off += (L.n_out * 4 + 15) / 16 * 16 + (L.n_out * pl->cell_bytes() + 15) / 16 * 16;
    }
    pl->side_bytes = off - (pl->total_cells * pl->cell_bytes() + 255) / 256 * 256;
  }
  pl->achieved_bits = 0;
  for (int l = 0; l < n_layers; ++l) {
    LayerGeom& L = pl->layers[l];
    L.cell_begin = pl->h_offsets[L.unit_begin];
    L.n_cells = pl->h_offsets[L.unit_begin + L.n_units] - L.cell_begin;
    int32_t mx = 0;
    for (int64_t u = L.unit_begin; u < L.unit_begin + L.n_units; ++u) mx = std::max(mx, pl->h_ncols[u]);
    L.max_ncols = mx;
    L.groups_one_n = 1;  // every key group of 8 units has one N (grouped-key build, query layout)
    for (int64_t u = 0; u < L.n_units && L.groups_one_n; u += kQGroup)
      for (int v = 1; v < kQGroup && u + v < L.n_units; ++v)
        if (pl->h_ncols[L.unit_begin + u + v] != pl->h_ncols[L.unit_begin + u]) {
          L.groups_one_n = 0;
          break;
        }
    L.achieved_bits = pl->q ? (L.n_cells + pl->G - 1) / pl->G * ((int64_t)pl->q * pl->G + 32) + L.meta_bits
                            : L.n_cells * state_bits + L.meta_bits + L.n_out * (32 + state_bits);
    pl->achieved_bits += L.achieved_bits;
  }
  if (pl->layout == USK_LAYOUT_QUERY) {
    s = qlayout_geometry(pl);
    if (s != USK_OK) {
      free_plan(pl);
      return s;
    }
  }
  *plan_out = pl;
  return USK_OK;
}

usk_status usk_plan_query(const usk_plan* pl, usk_plan_info* out) {
  if (!pl || !out) return fail(USK_EINVAL, "usk_plan_query: null");
  out->n_layers = pl->n_layers;
  out->rows = pl->M;
  out->n_classes = pl->C;
  out->dtype = pl->dtype;
  out->n_units = pl->U;
  out->total_cells = pl->total_cells;
  const int64_t bytes = pl->q ? pl->scales_off + pl->n_groups * 4
                              : (pl->total_cells * pl->cell_bytes() + 255) / 256 * 256 + pl->side_bytes;
  out->sketch_bytes = ((bytes + 255) / 256) * 256 + 256;
  if (pl->layout == USK_LAYOUT_QUERY) out->sketch_bytes = (pl->qtotal + 255) / 256 * 256 + 256;
  out->layout = pl->layout;
  out->hash = pl->hash_api;
  out->state_bits = pl->q;
  out->group_size = pl->q ? pl->G : 0;
  out->n_groups = pl->n_groups;
  out->scales_offset = pl->scales_off;
  out->topk = pl->topk;
  out->numel = pl->numel;
  out->budget_bits = pl->budget_bits;
  out->achieved_bits = pl->achieved_bits;
  return USK_OK;
}

usk_status usk_plan_layer(const usk_plan* pl, int32_t layer, usk_layer_info* out) {
  if (!pl || !out) return fail(USK_EINVAL, "usk_plan_layer: null");
  if (layer < 0 || layer >= pl->n_layers) return fail(USK_ESHAPE, "usk_plan_layer: layer out of range");
  const LayerGeom& L = pl->layers[layer];
  *out = usk_layer_info{L.out,         L.in,        L.unit_begin, L.n_units,       L.cell_begin, L.n_cells,
                        L.budget_bits, L.meta_bits, L.cells_T,    L.achieved_bits, L.n_out,      L.out_off,
                        L.qoff,        L.qbytes,    L.qmixed ? 0 : L.qcw};
  return USK_OK;
}

usk_status usk_plan_export(const usk_plan* pl, int32_t layer, uint8_t* cls, int32_t* ncols, uint8_t* nrows,
                           int64_t* offsets) {
  if (!pl) return fail(USK_EINVAL, "usk_plan_export: null plan");
  if (layer < 0 || layer >= pl->n_layers) return fail(USK_ESHAPE, "usk_plan_export: layer out of range");
  const LayerGeom& L = pl->layers[layer];
  if (cls) USK_CUDA(cudaMemcpy(cls, pl->d_cls + L.unit_begin, (size_t)L.n_units, cudaMemcpyDeviceToHost));
  if (ncols)
    USK_CUDA(cudaMemcpy(ncols, pl->d_ncols + L.unit_begin, sizeof(int32_t) * L.n_units, cudaMemcpyDeviceToHost));
  if (nrows) USK_CUDA(cudaMemcpy(nrows, pl->d_nrows + L.unit_begin, (size_t)L.n_units, cudaMemcpyDeviceToHost));
  if (offsets)
    USK_CUDA(cudaMemcpy(offsets, pl->d_offsets + L.unit_begin, sizeof(int64_t) * (L.n_units + 1),
                        cudaMemcpyDeviceToHost));
  return USK_OK;
}

usk_status usk_build_rows(const usk_plan* pl, int32_t layer, int64_t row_begin, int64_t row_end,
                          const void* weight_rows, void* sketch, usk_stream stream) {
  if (!pl || !weight_rows || !sketch) return fail(USK_EINVAL, "usk_build_rows: null pointer");
  if (!aligned16(sketch) || !aligned16(weight_rows)) return fail(USK_EINVAL, "usk_build_rows: 16-B alignment");
  if (pl->gran != USK_GRAN_OUTROW || pl->q) return fail(USK_EINVAL, "usk_build_rows: OUTROW plans with raw states");
  if (pl->layout != USK_LAYOUT_UNIT_MAJOR) return fail(USK_EUNSUPPORTED, "usk_build_rows: unit-major layout only");
  if (layer < 0 || layer >= pl->n_layers) return fail(USK_ESHAPE, "usk_build_rows: layer out of range");
  if (row_begin < 0 || row_end > pl->layers[layer].out || row_begin > row_end)
    return fail(USK_ESHAPE, "usk_build_rows: row range outside [0, out)");
  if (row_begin == row_end) return USK_OK;
  return launch_build_rows(pl, layer, row_begin, row_end, weight_rows, sketch, (cudaStream_t)stream);
}

usk_status usk_build(const usk_plan* pl, const void* const* weights, const int32_t* layer_ids, int32_t n,
                     void* sketch, usk_stream stream) {
  if (!pl || !weights || !sketch) return fail(USK_EINVAL, "usk_build: null pointer");
  if (!aligned16(sketch)) return fail(USK_EINVAL, "usk_build: sketch must be 16-B aligned");
  if (n < 0 || n > pl->n_layers) return fail(USK_ESHAPE, "usk_build: bad layer count");
  std::vector<char> seen(pl->n_layers, 0);
  for (int32_t k = 0; k < n; ++k) {
    const int32_t l = layer_ids ? layer_ids[k] : k;
    if (l < 0 || l >= pl->n_layers) return fail(USK_ESHAPE, "usk_build: layer id out of range");
    if (seen[l]) return fail(USK_EINVAL, "usk_build: duplicate layer id");
    seen[l] = 1;
    if (!weights[k]) return fail(USK_EINVAL, "usk_build: null weight pointer");
    if (!aligned16(weights[k])) return fail(USK_EINVAL, "usk_build: weights must be 16-B aligned");
  }
  if (pl->layout == USK_LAYOUT_QUERY) return launch_qbuild(pl, weights, layer_ids, n, sketch, (cudaStream_t)stream);
  return launch_build(pl, weights, layer_ids, n, sketch, (cudaStream_t)stream);
}

usk_status usk_reconstruct(const usk_plan* pl, const void* sketch, int32_t layer, int64_t row_begin, int64_t row_end,
                           void* w_out, int64_t ld_out, usk_stream stream) {
  if (!pl || !sketch || !w_out) return fail(USK_EINVAL, "usk_reconstruct: null pointer");
  if (layer < 0 || layer >= pl->n_layers) return fail(USK_ESHAPE, "usk_reconstruct: layer out of range");
  const LayerGeom& L = pl->layers[layer];
  if (row_begin < 0 || row_end > L.out || row_begin > row_end)
    return fail(USK_ESHAPE, "usk_reconstruct: row range outside [0, out_features)");
  if (ld_out < L.in) return fail(USK_ESHAPE, "usk_reconstruct: ld_out < in_features");
  if (pl->layout == USK_LAYOUT_QUERY)
    return launch_qreconstruct(pl, sketch, layer, row_begin, row_end, w_out, ld_out, (cudaStream_t)stream);
  return launch_reconstruct(pl, sketch, layer, row_begin, row_end, w_out, ld_out, (cudaStream_t)stream);
}

usk_status usk_reconstruct_batch(const usk_plan* pl, const void* sketch, const int32_t* layers, int32_t n,
                                 void* const* w_out, const int64_t* ld_out, usk_stream stream) {
  if (!pl || !sketch || !layers || !w_out || !ld_out) return fail(USK_EINVAL, "usk_reconstruct_batch: null pointer");
  if (n < 0) return fail(USK_ESHAPE, "usk_reconstruct_batch: n < 0");
  for (int32_t k = 0; k < n; ++k) {
    if (layers[k] < 0 || layers[k] >= pl->n_layers) return fail(USK_ESHAPE, "usk_reconstruct_batch: layer out of range");
    if (!w_out[k]) return fail(USK_EINVAL, "usk_reconstruct_batch: null w_out");
    if (ld_out[k] < pl->layers[layers[k]].in) return fail(USK_ESHAPE, "usk_reconstruct_batch: ld_out < in_features");
  }
  if (pl->layout == USK_LAYOUT_QUERY) return launch_qreconstruct_batch(pl, sketch, layers, n, w_out, ld_out, (cudaStream_t)stream);
  for (int32_t k = 0; k < n; ++k) {  // unit-major plans: one K3 launch per layer
    const LayerGeom& L = pl->layers[layers[k]];
    usk_status s = launch_reconstruct(pl, sketch, layers[k], 0, L.out, w_out[k], ld_out[k], (cudaStream_t)stream);
    if (s != USK_OK) return s;
  }
  return USK_OK;
}

usk_status usk_prefetch_l2(const usk_plan* pl, const void* sketch, int32_t layer_begin, int32_t layer_end,
                           usk_stream stream) {
  if (!pl || !sketch) return fail(USK_EINVAL, "usk_prefetch_l2: null pointer");
  if (layer_begin < 0 || layer_end > pl->n_layers || layer_begin > layer_end)
    return fail(USK_ESHAPE, "usk_prefetch_l2: layer range outside [0, n_layers)");
  return launch_prefetch(pl, sketch, layer_begin, layer_end, (cudaStream_t)stream);
}

size_t usk_linear_workspace_bytes(const usk_plan* pl, int32_t layer, int64_t T, int64_t out_begin,
                                  int64_t out_end) {
  if (!pl || layer < 0 || layer >= pl->n_layers || T < 1) return 0;
  const LayerGeom& L = pl->layers[layer];
  if (out_begin < 0 || out_end > L.out || out_begin > out_end) return 0;
  if (T == 1) {
    size_t b = pl->layout == USK_LAYOUT_QUERY ? qgemv_batch_workspace_bytes(pl, &layer, &out_begin, &out_end, 1)
                                              : gemv_workspace_bytes(pl, layer, out_begin, out_end);
    return b ? b : 256;
  }
  return (size_t)((out_end - out_begin) * L.in * 2 + 255) / 256 * 256;
}

usk_status usk_linear(const usk_plan* pl, const void* sketch, int32_t layer, const void* x, int32_t x_dtype,
                      int64_t T, void* y, int32_t y_dtype, int64_t out_begin, int64_t out_end, void* workspace,
                      size_t workspace_bytes, usk_stream stream) {
  if (!pl || !sketch || !x || !y) return fail(USK_EINVAL, "usk_linear: null pointer");
  if (x_dtype != USK_F32 && x_dtype != USK_BF16) return fail(USK_EINVAL, "usk_linear: x_dtype");
  if (y_dtype != USK_F32 && y_dtype != USK_BF16) return fail(USK_EINVAL, "usk_linear: y_dtype");
  if (!aligned16(x) || !aligned16(y) || !aligned16(sketch)) return fail(USK_EINVAL, "usk_linear: 16-B alignment");
  if (layer < 0 || layer >= pl->n_layers) return fail(USK_ESHAPE, "usk_linear: layer out of range");
  const LayerGeom& L = pl->layers[layer];
  if (T < 1) return fail(USK_ESHAPE, "usk_linear: T must be >= 1");
  if (out_begin < 0 || out_end > L.out || out_begin > out_end)
    return fail(USK_ESHAPE, "usk_linear: output range outside [0, out_features)");
  const size_t need = usk_linear_workspace_bytes(pl, layer, T, out_begin, out_end);
  if (workspace_bytes < need || (need && !workspace)) return fail(USK_ESHAPE, "usk_linear: workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  if (T == 1) {
    if (pl->layout == USK_LAYOUT_QUERY)
      return launch_qgemv_batch(pl, sketch, &layer, &out_begin, &out_end, 1, x, x_dtype, &y, y_dtype, workspace, st);
    return launch_gemv(pl, sketch, layer, x, x_dtype, y, y_dtype, out_begin, out_end, workspace, workspace_bytes, st);
  }
  if (pl->dtype != USK_BF16 || x_dtype != USK_BF16)
    return fail(USK_EUNSUPPORTED, "usk_linear: T > 1 needs bf16 weights and bf16 x (tcgen05 kind::f16)");
  const int64_t rows = out_end - out_begin;
  if (rows == 0) return USK_OK;
  if (!aligned16(workspace)) return fail(USK_EINVAL, "usk_linear: workspace alignment");
  // the paper's decompression: rebuild the output-row slice of W' ...
  usk_status s = pl->layout == USK_LAYOUT_QUERY
                     ? launch_qreconstruct(pl, sketch, layer, out_begin, out_end, workspace, L.in, st)
                     : launch_reconstruct(pl, sketch, layer, out_begin, out_end, workspace, L.in, st);
  if (s != USK_OK) return s;
  // ... then the computation stage on the tensor cores
  return launch_gemm_bf16(x, workspace, y, y_dtype, T, rows, L.in, L.in, st);
}

static usk_status batch_ranges(const usk_plan* pl, const int32_t* layers, const int64_t* ranges, int32_t n,
                               std::vector<int64_t>& o0, std::vector<int64_t>& o1) {
  if (!pl || !layers) return fail(USK_EINVAL, "usk_linear_batch: null pointer");
  if (n < 1 || n > 8) return fail(USK_ESHAPE, "usk_linear_batch: n must be in [1, 8]");
  o0.resize(n);
  o1.resize(n);
  for (int k = 0; k < n; ++k) {
    if (layers[k] < 0 || layers[k] >= pl->n_layers) return fail(USK_ESHAPE, "usk_linear_batch: layer out of range");
    const LayerGeom& L = pl->layers[layers[k]];
    if (L.in != pl->layers[layers[0]].in) return fail(USK_ESHAPE, "usk_linear_batch: in_features differ");
    o0[k] = ranges ? ranges[2 * k] : 0;
    o1[k] = ranges ? ranges[2 * k + 1] : L.out;
    if (o0[k] < 0 || o1[k] > L.out || o0[k] > o1[k])
      return fail(USK_ESHAPE, "usk_linear_batch: output range outside [0, out_features)");
  }
  return USK_OK;
}

static bool tokens_fused(const usk_plan* pl, const int32_t* layers, const std::vector<int64_t>& o0,
                         const std::vector<int64_t>& o1, int32_t n) {
  for (int k = 0; k < n; ++k) {
    const LayerGeom& L = pl->layers[layers[k]];
    if (o0[k] != 0 || o1[k] != L.out) return false;
    if (k + 1 < n && L.out % 32 != 0) return false;
  }
  return true;
}

size_t usk_linear_batch_tokens_workspace_bytes(const usk_plan* pl, const int32_t* layers, const int64_t* ranges,
                                               int32_t n, int64_t T) {
  if (T == 1) return usk_linear_batch_workspace_bytes(pl, layers, ranges, n);
  std::vector<int64_t> o0, o1;
  if (T < 1 || batch_ranges(pl, layers, ranges, n, o0, o1) != USK_OK) return 0;
  const int64_t in = pl->layers[layers[0]].in;
  int64_t rows = 0, mx = 0;
  for (int k = 0; k < n; ++k) {
    rows += o1[k] - o0[k];
    mx = std::max(mx, o1[k] - o0[k]);
  }
  return (size_t)(tokens_fused(pl, layers, o0, o1, n) ? rows : mx) * (size_t)in * 2;
}

usk_status usk_linear_batch_tokens(const usk_plan* pl, const void* sketch, const int32_t* layers,
                                   const int64_t* ranges, int32_t n, const void* x, int32_t x_dtype, int64_t T,
                                   void* const* y, int32_t y_dtype, void* workspace, size_t workspace_bytes,
                                   usk_stream stream) {
  if (T == 1)
    return usk_linear_batch(pl, sketch, layers, ranges, n, x, x_dtype, y, y_dtype, workspace, workspace_bytes,
                            stream);
  if (T < 1) return fail(USK_ESHAPE, "usk_linear_batch_tokens: T must be >= 1");
  std::vector<int64_t> o0, o1;
  usk_status s = batch_ranges(pl, layers, ranges, n, o0, o1);
  if (s != USK_OK) return s;
  if (!sketch || !x || !y || !workspace) return fail(USK_EINVAL, "usk_linear_batch_tokens: null pointer");
  if (y_dtype != USK_F32 && y_dtype != USK_BF16) return fail(USK_EINVAL, "usk_linear_batch_tokens: y_dtype");
  if (pl->dtype != USK_BF16 || x_dtype != USK_BF16)
    return fail(USK_EUNSUPPORTED, "usk_linear_batch_tokens: T > 1 needs bf16 weights and bf16 x (tcgen05 kind::f16)");
  if (!aligned16(x) || !aligned16(sketch) || !aligned16(workspace))
    return fail(USK_EINVAL, "usk_linear_batch_tokens: 16-B alignment");
  for (int k = 0; k < n; ++k)
    if (!y[k] || !aligned16(y[k])) return fail(USK_EINVAL, "usk_linear_batch_tokens: y pointer");
  if (workspace_bytes < usk_linear_batch_tokens_workspace_bytes(pl, layers, ranges, n, T))
    return fail(USK_ESHAPE, "usk_linear_batch_tokens: workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t in = pl->layers[layers[0]].in;
  unsigned char* ws = reinterpret_cast<unsigned char*>(workspace);
  if (!tokens_fused(pl, layers, o0, o1, n)) {  // one layer after another through the workspace
    for (int k = 0; k < n; ++k) {
      if (o1[k] == o0[k]) continue;
      s = pl->layout == USK_LAYOUT_QUERY ? launch_qreconstruct(pl, sketch, layers[k], o0[k], o1[k], ws, in, st)
                                         : launch_reconstruct(pl, sketch, layers[k], o0[k], o1[k], ws, in, st);
      if (s == USK_OK) s = launch_gemm_bf16(x, ws, y[k], y_dtype, T, o1[k] - o0[k], in, in, st);
      if (s != USK_OK) return s;
    }
    return USK_OK;
  }
  // decompression of the whole group (one launch on the query layout), then one GEMM
  std::vector<void*> wk(n);
  std::vector<int64_t> ld(n, in);
  std::vector<GemmOut> outs(n);
  int64_t row = 0;
  for (int k = 0; k < n; ++k) {
    wk[k] = ws + (size_t)row * in * 2;
    outs[k] = GemmOut{y[k], o1[k], o1[k]};
    row += o1[k];
  }
  if (pl->layout == USK_LAYOUT_QUERY) {
    s = launch_qreconstruct_batch(pl, sketch, layers, n, wk.data(), ld.data(), st);
  } else {
    for (int k = 0; k < n && s == USK_OK; ++k)
      s = launch_reconstruct(pl, sketch, layers[k], 0, o1[k], wk[k], in, st);
  }
  if (s != USK_OK) return s;
  return launch_gemm_bf16_seg(x, ws, outs.data(), n, y_dtype, T, in, st);
}

usk_status usk_gemm_tokens(const void* x, int64_t T, int64_t in, const void* w, const int64_t* rows, int32_t n,
                           void* const* y, int32_t y_dtype, usk_stream stream) {
  if (!x || !w || !rows || !y) return fail(USK_EINVAL, "usk_gemm_tokens: null pointer");
  if (n < 1 || n > 8 || T < 1 || in < 8 || in % 8 != 0) return fail(USK_ESHAPE, "usk_gemm_tokens: n, T or in");
  if (y_dtype != USK_F32 && y_dtype != USK_BF16) return fail(USK_EINVAL, "usk_gemm_tokens: y_dtype");
  if (!aligned16(x) || !aligned16(w)) return fail(USK_EINVAL, "usk_gemm_tokens: 16-B alignment");
  std::vector<GemmOut> outs(n);
  for (int k = 0; k < n; ++k) {
    if (rows[k] < 1 || (k + 1 < n && rows[k] % 32 != 0) || !y[k] || !aligned16(y[k]))
      return fail(USK_ESHAPE, "usk_gemm_tokens: rows[k] (inner blocks % 32 == 0) or y[k]");
    outs[k] = GemmOut{y[k], rows[k], rows[k]};
  }
  return launch_gemm_bf16_seg(x, w, outs.data(), n, y_dtype, T, in, (cudaStream_t)stream);
}

size_t usk_linear_batch_workspace_bytes(const usk_plan* pl, const int32_t* layers, const int64_t* ranges, int32_t n) {
  std::vector<int64_t> o0, o1;
  if (batch_ranges(pl, layers, ranges, n, o0, o1) != USK_OK) return 0;
  if (pl->layout == USK_LAYOUT_QUERY) return qgemv_batch_workspace_bytes(pl, layers, o0.data(), o1.data(), n);
  return gemv_batch_workspace_bytes(pl, layers, o0.data(), o1.data(), n);
}

usk_status usk_linear_batch(const usk_plan* pl, const void* sketch, const int32_t* layers, const int64_t* ranges,
                            int32_t n, const void* x, int32_t x_dtype, void* const* y, int32_t y_dtype, void* workspace,
                            size_t workspace_bytes, usk_stream stream) {
  std::vector<int64_t> o0, o1;
  usk_status s = batch_ranges(pl, layers, ranges, n, o0, o1);
  if (s != USK_OK) return s;
  if (!sketch || !x || !y || !workspace) return fail(USK_EINVAL, "usk_linear_batch: null pointer");
  if (x_dtype != USK_F32 && x_dtype != USK_BF16) return fail(USK_EINVAL, "usk_linear_batch: x_dtype");
  if (y_dtype != USK_F32 && y_dtype != USK_BF16) return fail(USK_EINVAL, "usk_linear_batch: y_dtype");
  if (!aligned16(x) || !aligned16(sketch) || !aligned16(workspace))
    return fail(USK_EINVAL, "usk_linear_batch: 16-B alignment");
  for (int k = 0; k < n; ++k)
    if (!y[k] || !aligned16(y[k])) return fail(USK_EINVAL, "usk_linear_batch: y pointer");
  if (pl->layout == USK_LAYOUT_QUERY) {
    if (workspace_bytes < qgemv_batch_workspace_bytes(pl, layers, o0.data(), o1.data(), n))
      return fail(USK_ESHAPE, "usk_linear_batch: workspace too small");
    return launch_qgemv_batch(pl, sketch, layers, o0.data(), o1.data(), n, x, x_dtype, y, y_dtype, workspace,
                              (cudaStream_t)stream);
  }
  if (workspace_bytes < gemv_batch_workspace_bytes(pl, layers, o0.data(), o1.data(), n))
    return fail(USK_ESHAPE, "usk_linear_batch: workspace too small");
  return launch_gemv_batch(pl, sketch, layers, o0.data(), o1.data(), n, x, x_dtype, y, y_dtype, workspace,
                           (cudaStream_t)stream);
}

usk_status usk_linear_batch_peers(const usk_plan* pl, const void* sketch, const int32_t* layers, const int64_t* ranges,
                                  int32_t n, const void* x, int32_t x_dtype, int32_t y_dtype, const usk_peers* peers,
                                  void* workspace, size_t workspace_bytes, usk_stream stream) {
  std::vector<int64_t> o0, o1;
  usk_status s = batch_ranges(pl, layers, ranges, n, o0, o1);
  if (s != USK_OK) return s;
  if (!peers || !sketch || !x || !workspace || !peers->y_peer || !peers->sig_peer || !peers->epoch)
    return fail(USK_EINVAL, "usk_linear_batch_peers: null pointer");
  if (pl->layout != USK_LAYOUT_QUERY) return fail(USK_EUNSUPPORTED, "usk_linear_batch_peers: query-layout plans only");
  if (peers->n_peers < 1 || peers->n_peers > 8 || peers->my_rank < 0 || peers->my_rank >= peers->n_peers)
    return fail(USK_EINVAL, "usk_linear_batch_peers: n_peers in [1, 8], 0 <= my_rank < n_peers");
  if (x_dtype != USK_F32 && x_dtype != USK_BF16) return fail(USK_EINVAL, "usk_linear_batch_peers: x_dtype");
  if (y_dtype != USK_F32 && y_dtype != USK_BF16) return fail(USK_EINVAL, "usk_linear_batch_peers: y_dtype");
  if (!aligned16(x) || !aligned16(sketch) || !aligned16(workspace))
    return fail(USK_EINVAL, "usk_linear_batch_peers: 16-B alignment");
  for (int q = 0; q < peers->n_peers; ++q) {
    if (!peers->sig_peer[q]) return fail(USK_EINVAL, "usk_linear_batch_peers: null signal pointer");
    for (int k = 0; k < n; ++k)
      if (!peers->y_peer[(size_t)q * n + k]) return fail(USK_EINVAL, "usk_linear_batch_peers: null y pointer");
  }
  if (workspace_bytes < qgemv_batch_workspace_bytes(pl, layers, o0.data(), o1.data(), n))
    return fail(USK_ESHAPE, "usk_linear_batch_peers: workspace too small");
  std::vector<void*> ymine(n);
  for (int k = 0; k < n; ++k) ymine[k] = peers->y_peer[(size_t)peers->my_rank * n + k];
  return launch_qgemv_batch(pl, sketch, layers, o0.data(), o1.data(), n, x, x_dtype, ymine.data(), y_dtype, workspace,
                            (cudaStream_t)stream, peers);
}

usk_status usk_peer_wait(const usk_plan* pl, const usk_peers* peers, usk_stream stream) {
  if (!pl || !peers || !peers->sig_peer || !peers->epoch) return fail(USK_EINVAL, "usk_peer_wait: null pointer");
  if (peers->n_peers < 1 || peers->n_peers > 8 || peers->my_rank < 0 || peers->my_rank >= peers->n_peers)
    return fail(USK_EINVAL, "usk_peer_wait: n_peers in [1, 8], 0 <= my_rank < n_peers");
  return launch_peer_wait(pl, peers, (cudaStream_t)stream);
}

usk_status usk_check(const usk_plan* pl, usk_stream stream) {
  if (!pl) return fail(USK_EINVAL, "usk_check: null plan");
  USK_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  int h = 0;
  USK_CUDA(cudaMemcpy(&h, pl->d_err, sizeof(int), cudaMemcpyDeviceToHost));
  if (h) {
    USK_CUDA(cudaMemset(pl->d_err, 0, sizeof(int)));
    if (h & 1) return fail(USK_ENONFINITE, "a build or aggregation saw NaN or Inf values");
    if (h & 4) return fail(USK_ECUDA, "usk_peer_wait: a peer rank never raised its flag (bounded spin expired)");
    return fail(USK_ERANGE, "a value of |v| >= 2^15 reached the 2^-48 fixed-point sums (CountMin / usk_aggregate_grad)");
  }
  return USK_OK;
}

void usk_plan_destroy(usk_plan* pl) { free_plan(pl); }

}  // extern "C"
