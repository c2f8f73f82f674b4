// grad.cu -- K8: the aggregated-gradient baseline of finetuning.
//
// §3.3 (Figure 4a): "Previous works estimate the gradient of trainable
// parameters by aggregating gradients from corresponding original weights".  Every weight adds
// its gradient to the cell it maps to in each sketch row; the sum is taken in 2^-48 fixed point
// with 64-bit integer atomics, so it is the same for every interleaving (DESIGN.md ledger L26).
// Not a hot path: one thread per weight, M global atomics each.
#include "common.cuh"

namespace usk {
namespace {

constexpr double kFix = 281474976710656.0;  // 2^48

struct AggArgs {
  const void* grad;
  int32_t bf16;
  int64_t out, in, unit_base, cell_begin;
  int32_t M, gran, g, hash;
  const int32_t* ncols;
  const uint8_t* nrows;  // M_u per unit (ledger L30)
  const int64_t* offsets;
  const uint32_t* ukeys;
  HashConsts hc;
  unsigned long long* acc;
  int* err;  // sticky flag: bit 0 non-finite value, bit 1 |value| >= 2^15 (outside the 2^-48 fixed point)
};

__global__ void k_aggregate(AggArgs A) {
  const int64_t n = A.out * A.in;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t o = e / A.in, j = e - o * A.in;
    int64_t t, p;
    unit_pos(A.gran, A.g, A.out, o, j, t, p);
    const int64_t u = A.unit_base + t;
    const uint32_t N = (uint32_t)A.ncols[u];
    const int64_t base = A.offsets[u] - A.cell_begin;
    const float gv = A.bf16 ? __uint_as_float((uint32_t)reinterpret_cast<const uint16_t*>(A.grad)[e] << 16)
                            : reinterpret_cast<const float*>(A.grad)[e];
    if (!isfinite(gv)) {  // q would saturate: flag it and leave it out of the sums
      atomicOr(A.err, 1);
      continue;
    }
    if (fabsf(gv) >= 32768.0f) atomicOr(A.err, 2);  // |q| >= 2^63: saturated, the sums are wrong
    const long long q = __double2ll_rn((double)gv * kFix);
    if (q == 0) continue;
    const uint32_t Ku = A.ukeys[u];
    const int Mu = A.nrows[u];
    for (int i = 0; i < Mu; ++i) {
      const uint32_t idx = A.hash == USK_HASH_X ? hash_index_x(A.hc, (uint32_t)p, Ku, i, N) : (uint32_t)(p % N);
      atomicAdd(&A.acc[base + (int64_t)i * N + idx], (unsigned long long)q);  // two's complement sum
    }
  }
}

__global__ void k_agg_finish(unsigned long long* acc, int64_t n, float* out) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= n) return;
  out[c] = __double2float_rn(__ll2double_rn((long long)acc[c]) * (1.0 / kFix));
  acc[c] = 0ull;  // leave the workspace zeroed
}

}  // namespace

size_t aggregate_workspace_bytes(const usk_plan* pl, int32_t l) {
  return (size_t)std::max<int64_t>(pl->layers[l].n_cells, 1) * 8;
}

// acc[c - cell_begin] += 2^-48 fixed point of vals (o, j) for every sketch row's cell of layer l
usk_status launch_fixed_accumulate(const usk_plan* pl, int32_t l, const void* vals, int32_t dtype,
                                   unsigned long long* acc, int* err, cudaStream_t st) {
  const LayerGeom& L = pl->layers[l];
  AggArgs A{vals, dtype == USK_BF16, L.out, L.in, L.unit_begin, L.cell_begin, pl->M, pl->gran, pl->g,
            pl->hash, pl->d_ncols, pl->d_nrows, pl->d_offsets, pl->d_keys, pl->hc, acc, err};
  const int64_t n = L.out * L.in;
  k_aggregate<<<(unsigned)std::min<int64_t>((n + 255) / 256, 148 * 32), 256, 0, st>>>(A);
  USK_LAUNCHED("k_aggregate");
  return USK_OK;
}

usk_status launch_aggregate(const usk_plan* pl, int32_t l, const void* grad, int32_t grad_dtype, float* cell_grad,
                            void* ws, cudaStream_t st) {
  const LayerGeom& L = pl->layers[l];
  usk_status s = launch_fixed_accumulate(pl, l, grad, grad_dtype, reinterpret_cast<unsigned long long*>(ws), pl->d_err,
                                         st);
  if (s != USK_OK) return s;
  struct {
    unsigned long long* acc;
  } A{reinterpret_cast<unsigned long long*>(ws)};
  if (L.n_cells > 0) {
    k_agg_finish<<<(unsigned)((L.n_cells + 255) / 256), 256, 0, st>>>(A.acc, L.n_cells, cell_grad);
    USK_LAUNCHED("k_agg_finish");
  }
  return USK_OK;
}

}  // namespace usk

using namespace usk;

extern "C" {

size_t usk_aggregate_grad_workspace_bytes(const usk_plan* pl, int32_t layer) {
  if (!pl || layer < 0 || layer >= pl->n_layers) return 0;
  return aggregate_workspace_bytes(pl, layer);
}

usk_status usk_aggregate_grad(const usk_plan* pl, int32_t layer, const void* grad, int32_t grad_dtype,
                              float* cell_grad, void* workspace, size_t workspace_bytes, usk_stream stream) {
  if (!pl || !grad || !cell_grad || !workspace) return fail(USK_EINVAL, "usk_aggregate_grad: null pointer");
  if (layer < 0 || layer >= pl->n_layers) return fail(USK_ESHAPE, "usk_aggregate_grad: layer out of range");
  if (grad_dtype != USK_F32 && grad_dtype != USK_BF16) return fail(USK_EINVAL, "usk_aggregate_grad: dtype");
  if (pl->q) return fail(USK_EUNSUPPORTED, "usk_aggregate_grad: raw-state plans only");
  if ((reinterpret_cast<uintptr_t>(workspace) & 15) != 0) return fail(USK_EINVAL, "workspace must be 16-B aligned");
  if (workspace_bytes < aggregate_workspace_bytes(pl, layer))
    return fail(USK_ESHAPE, "usk_aggregate_grad: workspace too small");
  return launch_aggregate(pl, layer, grad, grad_dtype, cell_grad, workspace, (cudaStream_t)stream);
}

}  // extern "C"
