// common.cuh -- shared internals of libusk (product path; independent of oracle/).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstring>

#include <string>
#include <vector>

#include "../../include/usk.h"

namespace usk {

// ----------------------------------------------------------------------------- errors
void set_error(const std::string& msg);
usk_status fail(usk_status st, const std::string& msg);
usk_status cuda_fail(cudaError_t e, const char* what);
void count_launch(int n = 1);
// cudaFuncSetAttribute once per (current device, kernel, attribute, value); thread-safe
cudaError_t ensure_func_attr(const void* kern, int attr, int value);
inline cudaError_t ensure_smem(const void* kern, int bytes) {
  return ensure_func_attr(kern, (int)cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}
int device_sm_count();  // SM count of the current device (cached per device)
unsigned long long* trace_slot(int grid);  // USK_TRACE ring slot of a launch (8 stamps per CTA) or nullptr

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
// USK-X (DESIGN.md 2.2 "Hash contract"; Eq. 3).  Host-side constants per
// sketch row i: rho_i = (u32) splitmix64(seed + 0x200 + i), kappa_i = (u32) splitmix64(seed + 0x300 + i);
// per unit K_u = (u32) splitmix64(seed ^ splitmix64((l << 32) | t)).  Per weight:
//   h_i = fmix32(p ^ rho_i) ^ fmix32(K_u ^ kappa_i)
//   idx_i = ((h_i mod 2^23) * N_u) >> 23 (N_u <= 2^16), else (h_i * N_u) >> 32.
// The fast kernels evaluate the short-unit reduction as one fp32 FMA rounded toward zero (see
// short_fma_bits); everything else calls hash_word / hash_reduce.
__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  uint64_t z = x;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// unit t (within its layer) and position p of weight (o, j) (L6/L31):
// ROW: t = j / g, p = (j - t g) out + o;  LAYER: t = 0, p = j out + o;  OUTROW: t = o, p = j
__host__ __device__ __forceinline__ void unit_pos(int32_t gran, int32_t g, int64_t out, int64_t o, int64_t j,
                                                  int64_t& t, int64_t& p) {
  if (gran == USK_GRAN_ROW) { t = j / g; p = (j - t * g) * out + o; }
  else if (gran == USK_GRAN_OUTROW) { t = o; p = j; }
  else { t = 0; p = j * out + o; }
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
  uint32_t rho[8];  // position salts rho_i
  uint32_t kap[8];  // unit-key salts kappa_i
};

constexpr uint32_t kShortUnitMax = 65536;  // N_u <= 2^16: 23-bit short-unit reduction

__host__ __device__ __forceinline__ uint32_t row_key(uint32_t Ku, uint32_t kap_i) { return fmix32(Ku ^ kap_i); }

__host__ __device__ __forceinline__ uint32_t hash_word(const HashConsts& hc, uint32_t p, uint32_t Ku, int i) {
  return fmix32(p ^ hc.rho[i]) ^ row_key(Ku, hc.kap[i]);
}

__host__ __device__ __forceinline__ uint32_t hash_reduce(uint32_t h, uint32_t N) {
  return N <= kShortUnitMax ? (uint32_t)(((uint64_t)(h & 0x7FFFFFu) * N) >> 23)
                            : (uint32_t)(((uint64_t)h * N) >> 32);
}

__host__ __device__ __forceinline__ uint32_t hash_index_x(const HashConsts& hc, uint32_t p, uint32_t Ku, int i,
                                                          uint32_t N) {
  return hash_reduce(hash_word(hc, p, Ku, i), N);
}

// Short-unit reduction in one FFMA.RZ: with f = as_float(0x3F800000 | k) =
// 1 + k / 2^23 and C = 2^25 - 4N + 4 off (off + N < 2^23), the exact f * 4N + C = 2^25 + 4 (off +
// k N / 2^23) lies in [2^25, 2^26) where the fp32 ulp is 4, so rounding toward zero gives
// 2^25 + 4 (off + floor(k N / 2^23)): the bit pattern 0x4C000000 + off + idx.  Biased exponent 152
// is a multiple of 4, so bits * 128 = (off + idx) * 128 mod 2^32: one IMAD to the shared address.
// fkey = 0x3F800000 | (row key mod 2^23); R23 = R_i mod 2^23; N4 = (float) 4N.
__device__ __forceinline__ uint32_t short_fma_bits(uint32_t R23, uint32_t fkey, float N4, uint32_t Cbits) {
  return __float_as_uint(__fmaf_rz(__uint_as_float(R23 ^ fkey), N4, __uint_as_float(Cbits)));
}
__host__ __device__ __forceinline__ uint32_t short_fkey(uint32_t rowkey) { return 0x3F800000u | (rowkey & 0x7FFFFFu); }
__host__ __device__ __forceinline__ uint32_t short_cbits(uint32_t N, uint32_t off) {
  // 2^25 - 4N + 4 off as fp32 bits (a multiple of 4 below 2^26: exact)
  const float c = (float)(int32_t)(33554432u - 4u * N + 4u * off);
#ifdef __CUDA_ARCH__
  return __float_as_uint(c);
#else
  uint32_t b;
  std::memcpy(&b, &c, 4);
  return b;
#endif
}

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
  int32_t groups_one_n = 0;  // every key group of 8 consecutive units has one N
  int32_t scope;      // budget scope id
  int64_t n_out = 0;  // Top-K outliers of the layer (L29)
  int64_t out_off = 0;  // byte offset of the layer's side table in the sketch (indices, then states)
  // query layout (usk.h USK_LAYOUT_QUERY): byte region of the layer, its first global chunk, chunks
  int64_t qoff = 0, qbytes = 0, qchunk0 = 0;
  int32_t qchunks = 0;
  int32_t qcw = 0;  // query layout: units per chunk of the layer's first chunk (256 / 128 / 64)
  int32_t qperm = 0;   // query layout: key groups in class order (importance classes, ledger L34)
  int32_t qmixed = 0;  // query layout: chunks of several widths
  struct QRun {        // maximal run of consecutive chunks of one width
    int32_t c0, n, cw;
  };
  std::vector<QRun> qruns;
};

constexpr int kQGroup = 8;  // units per key group (USK-XG, ledger L32) = cells per 16-B word of the query layout

}  // namespace usk

struct usk_plan {
  int32_t n_layers = 0, M = 3, gran = 0, g = 1, C = 1, min_cols = 1, hash = 0, dtype = 1;
  double bpw = 0;
  uint64_t seed = 0;
  int64_t U = 0, total_cells = 0, numel = 0, budget_bits = 0, achieved_bits = 0;
  int64_t max_out = 0;
  int64_t max_pos = 0;  // positions covered by d_R4: max over layers of max(out, in) (ROW: p = o, OUTROW: p = j)
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
  uint4* d_R4 = nullptr;       // {R_0, R_1, R_2} mod 2^23 per position p < max_pos (build bulk copies, K4o)
  int* d_err = nullptr;        // sticky device error flag
  int device = 0;
  // stacked state quantisation (L25): q = 0 (raw states) or 4 / 8 bits
  int32_t q = 0, G = 128;
  int32_t variant = 0;        // usk_variant (comparison variants: generic kernels only)
  std::vector<int32_t> Mc;    // sketch rows per class (ledger L30); M = max over the classes
  int64_t topk = 0;           // Top-K outliers per layer (0 = none)
  int64_t side_bytes = 0;     // bytes of all outlier side tables (after the cells)
  int64_t n_groups = 0;       // total_cells / G (quantised)
  int64_t scales_off = 0;     // byte offset of the fp32 group scales in the sketch (quantised)
  int32_t hash_api = 0;       // usk_hash as given; `hash` is the kernel family (USK-XG runs as USK-X: its
                              // grouped unit keys live in d_keys)
  int32_t layout = 0;         // usk_layout
  int64_t qtotal = 0;         // query layout: bytes of all layer regions
  std::vector<int64_t> h_qc_off;  // query layout: absolute byte offset of every chunk, [chunks + 1]
  std::vector<int32_t> h_qc_N;    //   and its maxN
  int64_t* d_qc_off = nullptr;
  int32_t* d_qc_N = nullptr;
  // per chunk (ledger L34): first query position (units, within the layer), units present, sketch rows,
  // width; per key group of the model: the layer-local group at each query position
  std::vector<int32_t> h_qc_q0, h_qc_n, h_qc_M, h_qc_cw, h_qperm;
  int32_t* d_qc_aux = nullptr;  // [4][chunks]: q0, n, M, cw
  int64_t* d_qc_lay = nullptr;  // [2][chunks]: the chunk's layer first unit; its first key group in
                                //   d_qperm for class-ordered layers, else -1 (k_qpack)
  int32_t* d_qperm = nullptr;   // [U / 8]
  int32_t* d_qg = nullptr;      // [2][U / 8]: each key group's query position (layer-local) and chunk
  int cell_bytes() const { return dtype == USK_BF16 ? 2 : 4; }  // raw state bytes
  int64_t code_bytes() const { return (total_cells * q + 7) / 8; }
};

namespace usk {
// launchers (defined in the .cu files)
usk_status launch_build(const usk_plan* pl, const void* const* weights, const int32_t* layer_ids,
                        int32_t n, void* sketch, cudaStream_t st);
usk_status launch_prefetch(const usk_plan* pl, const void* sketch, int32_t a, int32_t b, cudaStream_t st);
usk_status launch_build_rows(const usk_plan* pl, int32_t l, int64_t r0, int64_t r1, const void* w_rows, void* sketch,
                             cudaStream_t st);
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
// one GEMM over the concatenated W' rows of several layers, output columns split into segments
struct GemmOut {
  void* y;       // [T, cols] of the output dtype, leading dimension ld
  int64_t cols;  // inner segments: multiples of 32
  int64_t ld;
};
usk_status launch_gemm_bf16_seg(const void* X, const void* W, const GemmOut* outs, int nseg, int32_t y_dtype,
                                int64_t T, int64_t K, cudaStream_t st);
usk_status launch_importance(const void* A, int32_t a_dtype, int64_t N, int64_t d, float* I,
                             cudaStream_t st);
usk_status build_plan_device(usk_plan* pl, const float* const* saliency, cudaStream_t st);
usk_status launch_fixed_accumulate(const usk_plan* pl, int32_t l, const void* vals, int32_t dtype,
                                   unsigned long long* acc, int* err, cudaStream_t st);
bool layer_fast_ok(const usk_plan* pl, int32_t layer);
bool outrow_fast_ok(const usk_plan* pl, const int32_t* layers, int n);
// query layout (packed.cu)
usk_status qlayout_geometry(usk_plan* pl);
bool build_qfast_ok(const usk_plan* pl, const int32_t* layer_ids, int32_t n);
usk_status launch_build_qfast(const usk_plan* pl, const void* const* weights, const int32_t* layer_ids, int32_t n,
                              void* qsketch, cudaStream_t st);
usk_status launch_qbuild(const usk_plan* pl, const void* const* weights, const int32_t* layer_ids, int32_t n,
                         void* sketch, cudaStream_t st);
usk_status launch_qreconstruct(const usk_plan* pl, const void* sketch, int32_t layer, int64_t r0, int64_t r1,
                               void* w_out, int64_t ld, cudaStream_t st);
usk_status launch_qreconstruct_batch(const usk_plan* pl, const void* sketch, const int32_t* layers, int n,
                                     void* const* w_out, const int64_t* ld, cudaStream_t st);
size_t qgemv_batch_workspace_bytes(const usk_plan* pl, const int32_t* layers, const int64_t* o0, const int64_t* o1,
                                   int n);
usk_status launch_qgemv_batch(const usk_plan* pl, const void* sketch, const int32_t* layers, const int64_t* o0,
                              const int64_t* o1, int n, const void* x, int32_t x_dtype, void* const* y, int32_t y_dtype,
                              void* ws, cudaStream_t st, const usk_peers* peers = nullptr);
usk_status launch_peer_wait(const usk_plan* pl, const usk_peers* peers, cudaStream_t st);
usk_status launch_gemv_outrow(const usk_plan* pl, const void* sketch, const int32_t* layers, const int64_t* o0,
                              const int64_t* o1, int n, const void* x, int32_t x_dtype, void* const* y, int32_t y_dtype,
                              cudaStream_t st);
}  // namespace usk
