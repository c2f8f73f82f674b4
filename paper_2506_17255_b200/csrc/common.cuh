// common.cuh -- shared internals of libusk (product path; independent of oracle/).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include <string>
#include <vector>

#include "../../include/usk.h"

namespace usk {

// ----------------------------------------------------------------------------- errors
void set_error(const std::string& msg);
usk_status fail(usk_status st, const std::string& msg);
usk_status cuda_fail(cudaError_t e, const char* what);
void count_launch(int n = 1);

#define USK_CUDA(call)                                              \
  do {                                                              \
    cudaError_t _e = (call);                                        \
    if (_e != cudaSuccess) return ::usk::cuda_fail(_e, #call);      \
  } while (0)

#define USK_LAUNCHED(what)                                          \
  do {                                                              \
    cudaError_t _e = cudaGetLastError();                            \
    if (_e != cudaSuccess) return ::usk::cuda_fail(_e, what);       \
    ::usk::count_launch();                                          \
  } while (0)

// ----------------------------------------------------------------------------- hash contract
// USK-X (Eq. 3).  Host-side constants:
//   rho = (u32) splitmix64(seed); a_i = (u32) splitmix64(seed + 0x100 + i) | 1;
//   K_u = (u32) splitmix64(seed ^ splitmix64((l << 32) | t)).
// Device side per weight:  idx_i = mulhi32((fmix32(p ^ rho) ^ K_u) * a_i, N_u).
__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  uint64_t z = x;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__host__ __device__ __forceinline__ uint32_t fmix32(uint32_t h) {
  h ^= h >> 16;
  h *= 0x85EBCA6Bu;
  h ^= h >> 13;
  h *= 0xC2B2AE35u;
  h ^= h >> 16;
  return h;
}

struct HashConsts {
  uint32_t rho;
  uint32_t a[8];
};

// Key encodings on 32-bit words (weights held with their bits in the HIGH position: bf16
// bits << 16, fp32 bits as-is).  With mag = magnitude bits and s = sign bit:
//   kappa = rotl(b, 1) = (mag << 1) | s        -- build order: min kappa = min |w|, tie -> +
//   rho   = kappa ^ 1  = (mag << 1) | (1 - s)  -- retrieve order: max rho = max |w|, tie -> +
//   rotr(rho, 1)       = bits of -w            -- so x * w = (-x) * rotr(rho, 1)
// Empty build key = 0xFFFFFFFF (decodes to +Inf state).
__device__ __forceinline__ uint32_t rotl1(uint32_t v) { return __funnelshift_l(v, v, 1); }
__device__ __forceinline__ uint32_t rotr1(uint32_t v) { return __funnelshift_r(v, v, 1); }

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ----------------------------------------------------------------------------- plan
struct LayerGeom {
  int64_t out, in;
  int64_t unit_begin, n_units;
  int64_t cell_begin, n_cells;
  int64_t budget_bits, meta_bits, cells_T, achieved_bits;
  int32_t max_ncols;  // max N over the layer's units
  int32_t scope;      // budget scope id
  int64_t n_out = 0;  // Top-K outliers of the layer (L29)
  int64_t out_off = 0;  // byte offset of the layer's side table in the sketch (indices, then states)
};

}  // namespace usk

struct usk_plan {
  int32_t n_layers = 0, M = 3, gran = 0, g = 1, C = 1, min_cols = 1, hash = 0, dtype = 1;
  double bpw = 0;
  uint64_t seed = 0;
  int64_t U = 0, total_cells = 0, numel = 0, budget_bits = 0, achieved_bits = 0;
  int64_t max_out = 0;
  usk::HashConsts hc{};
  std::vector<usk::LayerGeom> layers;
  std::vector<int32_t> h_ncols;    // [U]
  std::vector<int64_t> h_offsets;  // [U+1]
  std::vector<uint8_t> h_cls;      // [U]
  // device
  uint8_t* d_cls = nullptr;
  int32_t* d_ncols = nullptr;
  uint8_t* d_nrows = nullptr;
  int64_t* d_offsets = nullptr;
  uint32_t* d_keys = nullptr;  // K_u per unit
  uint32_t* d_R = nullptr;     // R(o) = fmix32(o ^ rho), o < max_out (g = 1 positions)
  int* d_err = nullptr;        // sticky device error flag
  int device = 0;
  // stacked state quantisation (L25): q = 0 (raw states) or 4 / 8 bits
  int32_t q = 0, G = 128;
  int32_t variant = 0;        // usk_variant (comparison variants: generic kernels only)
  int64_t topk = 0;           // Top-K outliers per layer (0 = none)
  int64_t side_bytes = 0;     // bytes of all outlier side tables (after the cells)
  int64_t n_groups = 0;       // total_cells / G (quantised)
  int64_t scales_off = 0;     // byte offset of the fp32 group scales in the sketch (quantised)
  int cell_bytes() const { return dtype == USK_BF16 ? 2 : 4; }  // raw state bytes
  int64_t code_bytes() const { return (total_cells * q + 7) / 8; }
};

namespace usk {
// launchers (defined in the .cu files)
usk_status launch_build(const usk_plan* pl, const void* const* weights, const int32_t* layer_ids,
                        int32_t n, void* sketch, cudaStream_t st);
usk_status launch_reconstruct(const usk_plan* pl, const void* sketch, int32_t layer, int64_t r0,
                              int64_t r1, void* w_out, int64_t ld, cudaStream_t st);
usk_status launch_gemv(const usk_plan* pl, const void* sketch, int32_t layer, const void* x,
                       int32_t x_dtype, void* y, int32_t y_dtype, int64_t o0, int64_t o1,
                       void* ws, size_t ws_bytes, cudaStream_t st);
size_t gemv_workspace_bytes(const usk_plan* pl, int32_t layer, int64_t o0, int64_t o1);
size_t gemv_batch_workspace_bytes(const usk_plan* pl, const int32_t* layers, const int64_t* o0, const int64_t* o1,
                                  int n);
usk_status launch_gemv_batch(const usk_plan* pl, const void* sketch, const int32_t* layers, const int64_t* o0,
                             const int64_t* o1, int n, const void* x, int32_t x_dtype, void* const* y, int32_t y_dtype,
                             void* ws, cudaStream_t st);
usk_status launch_gemm_bf16(const void* X, const void* W, void* Y, int32_t y_dtype, int64_t T,
                            int64_t n_out, int64_t K, int64_t ldw, cudaStream_t st);
usk_status launch_importance(const void* A, int32_t a_dtype, int64_t N, int64_t d, float* I,
                             cudaStream_t st);
usk_status build_plan_device(usk_plan* pl, const float* const* saliency, cudaStream_t st);
usk_status launch_fixed_accumulate(const usk_plan* pl, int32_t l, const void* vals, int32_t dtype,
                                   unsigned long long* acc, int* err, cudaStream_t st);
bool layer_fast_ok(const usk_plan* pl, int32_t layer);
}  // namespace usk
