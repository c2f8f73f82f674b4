/*
 * usk.h -- C ABI of the B200-native UltraSketchLLM sketch engine (arXiv 2506.17255).
 *
 * The library implements the paper's index-free multi-row AbsMaxMin sketch hot path on
 * sm_100a: importance-aware space allocation (§3.4), the sketch build (§3.2 select/update,
 * §3.5 "AbsMin Scatter operator"), and the query fused into the consuming linear layer
 * (§3.1 decompression -> computation; §3.5 "modify the linear layer correspondingly").
 *
 * Conventions (all entry points):
 *   - Plain pointers and sizes only.  "device" = CUDA device memory of the current device;
 *     "host" = ordinary host memory.  Every large buffer is CALLER-OWNED.
 *   - The plan is an opaque, library-owned, immutable handle (usk_plan_destroy frees it).
 *   - usk_reconstruct / usk_linear never allocate; usk_build / usk_build_rows take only
 *     stream-ordered temporaries (cudaMallocAsync: the raw states of quantised plans, the
 *     transposed weights of output-row units).  All are asynchronous on `stream` (NULL = legacy
 *     default stream) and may run concurrently on different streams with one plan.  usk_plan_allocation synchronises `stream` once (launch geometry lives on host).
 *   - Return USK_OK (0) or an error code; no exception or abort crosses the ABI.  A one-line
 *     diagnostic of the last failure on the calling thread is in usk_last_error().
 *   - Results are a pure function of the inputs: sketch bytes and reconstructions do not
 *     depend on launch configuration, stream, GPU count or thread interleaving
 *     (order independence); usk_linear is deterministic for fixed inputs.
 *
 * Citations: PAPER.md:<line> (section / equation).  Readings where the paper is silent are
 * listed in DESIGN.md ("ledger" L1..L34) and referenced below.
 */
#ifndef USK_H
#define USK_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define USK_API __attribute__((visibility("default")))
#else
#define USK_API
#endif

typedef struct CUstream_st* usk_stream; /* == cudaStream_t */

typedef enum {
  USK_OK = 0,
  USK_EINVAL = 1,       /* null pointer, bad enum, rows not in [1,8], bpw <= 0 or non-finite,
                           dims_per_unit does not divide in_features, negative / NaN saliency,
                           misaligned pointer (16 B required for x, y, weights, sketch, w_out) */
  USK_ESHAPE = 2,       /* zero-size layer, layer id / row range / output range out of bounds,
                           count mismatch, workspace too small */
  USK_EBUDGET = 3,      /* infeasible floor: sum_c n_c * M * min_cols > T cells */
  USK_ENONFINITE = 4,   /* the build saw NaN or +-Inf (sticky; reported by usk_check) --
                           +Inf is the empty-cell sentinel (L4) */
  USK_ECUDA = 5,        /* CUDA launch / runtime failure (text in usk_last_error) */
  USK_EUNSUPPORTED = 6, /* valid request with no kernel (e.g. T > 1 with fp32 weights) */
  USK_ERANGE = 7        /* a value of |v| >= 2^15 entered a 2^-48 fixed-point sum (CountMin build,
                           usk_aggregate_grad; L26/L27): the affected sums saturated
                           (sticky; reported by usk_check) */
} usk_status;

typedef enum { USK_F32 = 0, USK_BF16 = 1 } usk_dtype;

/* Sketch-space granularity: ROW = one sketch per input dimension of a
 * weight matrix (per `dims_per_unit` input dims; L6/L7); LAYER = one per matrix;
 * OUTROW = one per OUTPUT row o of the [out, in] matrix, positions p = j ("each row
 * of the weight matrix corresponds to an independent AbsMaxMin sketch instance"; L31).
 * OUTROW units all carry the layer's mean saliency, so they form one class (n_classes 0 or 1);
 * dims_per_unit must be 1.  Its decode runs one kernel per call (no cross-CTA reduction). */
typedef enum { USK_GRAN_ROW = 0, USK_GRAN_LAYER = 1, USK_GRAN_OUTROW = 2 } usk_granularity;

/* Hash family (Eq. 3; contract in DESIGN.md 2.2 "Hash contract USK-X"):
 * USK_HASH_X = per-row salted position mix fmix32(p ^ rho_i) XOR per-unit key fmix32(K_u ^ kappa_i),
 * reduced to [0, N_u) by the top 23 bits times N_u (short units, N_u <= 2^16; exact as one fp32
 * FMA.RZ on the device) or a 32-bit multiply-high (long units); USK_HASH_IDENTITY = p mod N
 * (tests only). */
typedef enum { USK_HASH_X = 0, USK_HASH_IDENTITY = 1, USK_HASH_XG = 2 } usk_hash;
/* USK_HASH_XG (DESIGN.md ledger L32): USK-X with the unit key of the KEY GROUP floor(t / 8) -- the
 * 8 consecutive units t = 8g .. 8g+7 of a layer share the M functions H_i of PAPER.md:239-243
 * ("I = H(Addr(w))", one set of independent H_0..H_{M-1} of the weight's bias), groups use
 * independent ones.  Required by the query layout below. */

/* Sketch storage layout.
 * USK_LAYOUT_UNIT_MAJOR (default): the cells of unit u at [offsets[u], offsets[u+1]) in the state
 *   dtype, row-major (i, c) inside the unit (usk_plan_export).
 * USK_LAYOUT_QUERY (round 2; bf16 states, ROW units with dims_per_unit 1, USK_HASH_XG, AbsMaxMin,
 *   raw states, no Top-K, in_features % 8 == 0, every key group of 8 units with one N, a 64-unit
 *   chunk's M_k * maxN_k * 128 bytes within the chunk budget of 226,240 bytes, and the chunks' padding of existing units
 *   (N_u < maxN_k or M_u < M_k) at most 1/16 of each layer's cells): the same cells, permuted and
 *   re-encoded for the decode so that one 16-, 8- or 4-byte shared load gathers a lane's 8, 4 or 2
 *   cells of a sketch row (DESIGN.md §4 / §5 K4p, ledger L32, L34).  Each layer occupies
 *   [qbyte_begin, qbyte_begin + qbytes) (usk_layer_info).
 *   Query order of a layer: its key groups (units 8g .. 8g+7) in order of the class of their units
 *   (usk_plan_export cls; stable, so by g inside a class) -- the identity when all groups share a
 *   class; query position q is unit 8 * group(q / 8) + q % 8.
 *   Chunks cover consecutive query positions from 0: a chunk starts where the previous ends and
 *   takes CW_k positions, cut short at the layer end and, when the layer has several classes, at the
 *   next class boundary.  CW_k = 256 when M_k * maxN_k * 512 <= 226,240 bytes, else 128,
 *   else 64 (maxN_k, M_k: the largest N_u and sketch rows M_u of the chunk's units); a layer with one
 *   class takes one CW for all its chunks, from its largest M_u and N_u (usk_layer_info
 *   qchunk_units; 0 when a layer's chunks have several widths).  Chunk k takes
 *   M_k * maxN_k * 2 * CW_k bytes (the chunk's whole width, present units or not), chunks back to
 *   back from qbyte_begin.  Inside chunk k, the 16-bit word at byte
 *       ((i * maxN_k + c) * CW_k + s) * 2
 *   holds cell (i, c) of the unit at query position q0_k + s as the retrieve key
 *       rho16 = ((b << 1) | (b >> 15)) ^ 1  (b = the bf16 bits of the state; mag << 1 | 1 - sign),
 *   and 0 where the position is past the chunk's units, c >= N_u or i >= M_u (0 is below every key:
 *   neutral for the Eq. 5 max). */
typedef enum { USK_LAYOUT_UNIT_MAJOR = 0, USK_LAYOUT_QUERY = 1 } usk_layout;

/* Sketch variant (Appendix C.2): USK_ABSMAXMIN = the paper's sketch (keep the
 * min |.|, retrieve the max |.|); USK_ABSMINMAX = the order of min and max swapped (cells start at
 * +0); USK_COUNTMIN = cells hold the sum of their weights (2^-48 fixed point, ledger L26/L27),
 * retrieve the min |.|.  Ties prefer the non-negative value in every variant. */
typedef enum { USK_ABSMAXMIN = 0, USK_ABSMINMAX = 1, USK_COUNTMIN = 2 } usk_variant;

/* One linear layer, PyTorch layout: weight is row-major [out_features, in_features]. */
typedef struct {
  int64_t out_features;
  int64_t in_features;
} usk_shape;

typedef struct {
  double bpw;            /* budget in bits per weight (Table 1 "Equivalent Bits", PAPER.md:376;
                            states are raw, L3) */
  int32_t rows;          /* M, sketch rows, [1, 8]; paper default 3 */
  int32_t granularity;   /* usk_granularity */
  int32_t dims_per_unit; /* g >= 1, ROW only; must divide in_features (L7) */
  int32_t n_classes;     /* C >= 1 importance categories; 0 = default
                            (4 when saliency is given, else 1) */
  int32_t min_cols;      /* floor of columns per row, >= 1 (L12) */
  int32_t hash;          /* usk_hash */
  int32_t dtype;         /* usk_dtype of weights == dtype of sketch states (L3) */
  uint64_t seed;         /* hash seed ("fixing random seed in hash functions") */
  int32_t state_bits;    /* 0: raw states in the weight dtype; 4 or 8: stacked state quantisation
                            (Table 1 "+ q4"/"+ q8"): codes of
                            state_bits bits, one fp32 absmax scale per group_size cells of a layer,
                            round half away from zero; DESIGN.md ledger L25 */
  int32_t group_size;    /* cells per scale group (power of two >= 32; 0 = 128); quantised plans only */
  int32_t variant;       /* usk_variant: the sketch (Appendix C.2; L27).
                            The comparison variants run on the generic kernels, raw states only. */
  const double* layer_importance; /* host [n_layers] >= 0, or NULL.  Non-NULL (ROW granularity, raw
                            states): two-level allocation -- one model budget floor(bpw * numel),
                            split over layers in proportion to importance_l * numel_l (2^24 fixed
                            point, water-filled floors U_l * M * min_cols, largest remainder), then
                            the row allocation inside each layer (L28).
                            NULL: every layer is its own budget scope. */
  int64_t topk;          /* Top-K outliers per layer (App. A): the min(topk, numel)
                            weights of largest |w| (ties -> smaller flat index o*in + j) are kept
                            exactly in a side table of (int32 flat index, state) pairs charged to
                            the layer budget (32 + state bits each), left out of the sketch, and
                            overlaid on every retrieval (L29).  ROW granularity, raw
                            states, AbsMaxMin only; 0 = none. */
  const int32_t* class_rows; /* host [n_classes] sketch rows per importance class, each in [1, 8], or
                            NULL (every class has `rows`).  The north star's "salient weights more
                            rows or buckets" (categories PAPER.md:523-528; DESIGN.md
                            L30): class c's share of the cells (proportional to its importance, as
                            without class_rows) is laid out as class_rows[c] rows of N_c columns,
                            x_c = T W_c / (W n_c class_rows[c]).  Unit u has M_u = class_rows[cls_u]
                            rows (usk_plan_export nrows); usk_plan_info.rows = max_c class_rows[c].
                            AbsMaxMin only; not with layer_importance. */
  int32_t layout;        /* usk_layout of the sketch buffer (USK_LAYOUT_UNIT_MAJOR = 0 by default).
                            USK_LAYOUT_QUERY: usk_build writes the query layout, usk_reconstruct /
                            usk_linear / usk_linear_batch / usk_prefetch_l2 read it; usk_stats,
                            usk_aggregate_grad and usk_build_rows return USK_EUNSUPPORTED.  A plan
                            that does not meet the layout's conditions fails with USK_EUNSUPPORTED. */
  int32_t reserved;
} usk_params;

typedef struct usk_plan usk_plan;

typedef struct {
  int32_t n_layers;
  int32_t rows;
  int32_t n_classes;
  int32_t dtype;
  int64_t n_units;
  int64_t total_cells;    /* sum over units of M * N_u */
  int64_t sketch_bytes;   /* bytes the caller must allocate for the sketch (cells + tail pad) */
  int64_t numel;          /* weights covered */
  int64_t budget_bits;    /* sum of floor(bpw * numel) over budget scopes */
  int64_t achieved_bits;  /* states * state bits + charged class-map bits (<= budget_bits);
                             quantised: sum over layers of ceil(cells/G) * (q*G + 32) + class map */
  int32_t state_bits;     /* 0 (raw), 4 or 8 */
  int32_t group_size;     /* quantised plans: cells per scale group */
  int64_t n_groups;       /* quantised plans: total_cells / group_size (layers start at multiples
                             of group_size, total_cells includes the padding) */
  int64_t scales_offset;  /* quantised plans: byte offset of the fp32 scales in the sketch buffer;
                             the codes (packed, cell c at bit c*state_bits) start at byte 0 */
  int64_t topk;           /* Top-K outliers per layer (0 = none) */
  int32_t layout;         /* usk_layout of the sketch buffer */
  int32_t hash;           /* usk_hash */
} usk_plan_info;

typedef struct {
  int64_t out_features;
  int64_t in_features;
  int64_t unit_begin;     /* first global unit id of the layer */
  int64_t n_units;
  int64_t cell_begin;     /* first cell of the layer in the sketch */
  int64_t n_cells;
  int64_t budget_bits;    /* ROW: floor(bpw * numel_l); LAYER: model budget on layer 0, else 0 */
  int64_t meta_bits;      /* charged class-map bits (ROW with C > 1: U_l * ceil(log2 C)) */
  int64_t cells_T;        /* cells available to the scope (ROW per layer; LAYER on layer 0) */
  int64_t achieved_bits;  /* states of this layer * state bits + meta_bits (+ outlier side table) */
  int64_t n_outliers;     /* Top-K: outliers of this layer (min(topk, numel)) */
  int64_t outlier_offset; /* Top-K: byte offset in the sketch of the layer's side table: n_outliers
                             int32 flat indices (ascending), then at the next 16-B boundary their
                             states in the plan dtype */
  int64_t qbyte_begin;    /* USK_LAYOUT_QUERY: byte offset of the layer's region in the sketch */
  int64_t qbytes;         /*   and its size (0 for the unit-major layout) */
  int32_t qchunk_units;   /*   units per chunk CW (256, 128 or 64); 0 when the layer mixes widths */
  int32_t reserved;
} usk_layer_info;

/* Importance metric, Eq. 7: I[j] = (1/N) sum_k A[k, j]^2.
 * A: device, row-major [N, d] of dtype a_dtype (USK_F32 or USK_BF16); I_out: device float[d].
 * fp32 accumulation in a fixed order (deterministic).  Errors: EINVAL (null, dtype), ESHAPE
 * (N < 1 or d < 1), ECUDA. */
USK_API usk_status usk_importance(const void* A, int32_t a_dtype, int64_t N, int64_t d, float* I_out,
                          usk_stream stream);

/* Salient-weight-aware sketch space allocation (§3.4; categories
 * PAPER.md:523-528), computed on the device: per-unit scores -> 2^24 fixed point -> rank ->
 * equal-count classes -> per-class columns (proportional share, water-filled floor, largest
 * remainder) -> device-wide exclusive prefix scan of unit sizes.
 *   layers:   host array [n_layers] of shapes; list position = hash layer id.
 *   saliency: host array [n_layers] of DEVICE pointers to float[in_features] scores (>= 0),
 *             or NULL (uniform).  An individual NULL entry means uniform for that layer.
 *   params:   host.
 *   plan_out: receives the new plan.  On error *plan_out is NULL.
 * Synchronises `stream`.  Errors: EINVAL, ESHAPE, EBUDGET, ECUDA. */
USK_API usk_status usk_plan_allocation(const usk_shape* layers, int32_t n_layers,
                               const float* const* saliency, const usk_params* params,
                               usk_plan** plan_out, usk_stream stream);

USK_API usk_status usk_plan_query(const usk_plan* plan, usk_plan_info* out);
USK_API usk_status usk_plan_layer(const usk_plan* plan, int32_t layer, usk_layer_info* out);

/* Host copies of one layer's plan arrays (parity tests): cls[n_units], ncols[n_units],
 * nrows[n_units], offsets[n_units + 1] (absolute cells).  Any output may be NULL.  Syncs. */
USK_API usk_status usk_plan_export(const usk_plan* plan, int32_t layer, uint8_t* cls, int32_t* ncols,
                           uint8_t* nrows, int64_t* offsets);

/* Build (§3.2: select Eq. 3, update Eq. 4; "AbsMin Scatter"):
 *   S[u, i, c] = the colliding weight of minimum |.| (ties -> non-negative, L2),
 *   +Inf when no weight maps to the cell.
 *   weights:   host array [n] of DEVICE pointers, weights[k] = row-major [out, in] of the plan
 *              dtype for layer layer_ids[k].
 *   layer_ids: host int32[n], distinct, or NULL = layers 0..n-1 (layer-sharded builds pass a
 *              subset; only those layers' cells are written).
 *   sketch:    device, >= sketch_bytes, 16-B aligned; cells of layer l at
 *              [cell_begin, cell_begin + n_cells), unit-major, row-major (i, c) inside a unit.
 * Non-finite weights set the plan's sticky flag (usk_check -> USK_ENONFINITE). */
USK_API usk_status usk_build(const usk_plan* plan, const void* const* weights, const int32_t* layer_ids,
                     int32_t n, void* sketch, usk_stream stream);

/* Row-sharded build of OUTPUT-ROW units (USK_GRAN_OUTROW, L31; SURVEY 8(f4) "disjoint
 * per-rank sketch shards"): writes only the cells of the units of output rows [row_begin, row_end)
 * of `layer` -- byte-identical to those usk_build writes -- so the ranks of an output-sharded
 * deployment each build and keep just their own rows, with no sketch replication.
 *   weight_rows: device, the rows [row_begin, row_end) of the layer's [out, in] matrix (row-major,
 *                leading dimension in_features; rows outside the range are not needed), 16-B aligned.
 * USK_EINVAL unless the plan is OUTROW with raw states (quantisation groups span rows); USK_ESHAPE
 * for a bad layer / row range; USK_EUNSUPPORTED when the layer is not eligible for the fast build
 * (AbsMaxMin, in_features * state bytes a multiple of 16, slots within shared memory). */
USK_API usk_status usk_build_rows(const usk_plan* plan, int32_t layer, int64_t row_begin, int64_t row_end,
                          const void* weight_rows, void* sketch, usk_stream stream);

/* Reconstruction / decompression (Eq. 5; §3.1):
 *   w'(o, j) = the bonded cell of maximum |.| over the M rows (ties -> non-negative, L1/L2).
 *   Writes rows [row_begin, row_end) of W' (output features) as a row-major device matrix of
 *   the plan dtype with leading dimension ld_out (elements, >= in_features) at w_out. */
USK_API usk_status usk_reconstruct(const usk_plan* plan, const void* sketch, int32_t layer,
                           int64_t row_begin, int64_t row_end, void* w_out, int64_t ld_out,
                           usk_stream stream);

/* Reconstruction of whole layers, several per launch (query layout: consecutive layers with one
 * in_features share K3p launches, one per chunk width present, up to 8 layers; unit-major: one
 * launch per layer):
 * layer layers[k] into w_out[k] (device, row-major [out, in] of the plan dtype, leading dimension
 * ld_out[k] >= in_features).  Same bytes as usk_reconstruct of each layer. */
USK_API usk_status usk_reconstruct_batch(const usk_plan* plan, const void* sketch, const int32_t* layers, int32_t n,
                                         void* const* w_out, const int64_t* ld_out, usk_stream stream);

/* L2 warm-up of the sketch bytes of layers [layer_begin, layer_end) (cells, or codes + group
 * scales of a quantised plan, and their Top-K side tables): bulk L2 prefetches issued by a small
 * grid launched with programmatic dependent launch, so it overlaps the running kernel; the
 * following usk_linear calls then stage their chunks from L2 instead of HBM.  A pure performance
 * hint: no results change.  Stream-ordered after the previous work on `stream` (the kernel waits
 * for its predecessor before it completes).  Use it where the sketch region fits L2 (126 MB on
 * B200), e.g. once per decode token for a 1B model (60 MB), or one block ahead for larger ones.
 *   USK_ESHAPE for a layer range outside [0, n_layers); USK_EINVAL for null pointers. */
USK_API usk_status usk_prefetch_l2(const usk_plan* plan, const void* sketch, int32_t layer_begin,
                                   int32_t layer_end, usk_stream stream);

/* Workspace bytes usk_linear needs for (layer, T, output range).  0 on invalid arguments. */
USK_API size_t usk_linear_workspace_bytes(const usk_plan* plan, int32_t layer, int64_t T,
                                  int64_t out_begin, int64_t out_end);

/* Sketch-fused linear (PAPER.md:183-189 decompress -> compute; §3.5 modified linear):
 *   y[t, o - out_begin] = sum_j x[t, j] * w'(o, j),  o in [out_begin, out_end), t < T.
 *   x: device [T, in_features] of x_dtype; y: device [T, out_end - out_begin] of y_dtype.
 *   T == 1 : sketch-GEMV, W' rebuilt in registers and never stored; fp32 accumulation and a
 *            fixed-order split-K reduction (deterministic).  Launched with programmatic
 *            dependent launch: x may be produced by the previous kernel on the stream.
 *   T >  1 : bf16 plans and bf16 x only -- W' rows rebuilt into `workspace` (the paper's
 *            decompression), then a tcgen05 tensor-core GEMM with fp32 accumulation.
 *   workspace: device, >= usk_linear_workspace_bytes(...), 16-B aligned; MUST be zero-filled
 *   before its first use -- every call leaves it zero-filled again. */
USK_API usk_status usk_linear(const usk_plan* plan, const void* sketch, int32_t layer, const void* x,
                      int32_t x_dtype, int64_t T, void* y, int32_t y_dtype, int64_t out_begin,
                      int64_t out_end, void* workspace, size_t workspace_bytes,
                      usk_stream stream);

/* Several sketch-GEMVs that share one input vector in ONE launch (q|k|v, gate|up of a
 * transformer block): for k < n,
 *   y[k][o - ranges[2k]] = sum_j x[j] * w'_{layers[k]}(o, j),  o in [ranges[2k], ranges[2k+1]).
 *   layers: host int32[n] (n <= 8), all with the same in_features; ranges: host int64[2n] or NULL
 *   (full output range); x: device [in] (T = 1); y: host array of n device pointers.
 *   Same numerics as n calls of usk_linear (T = 1).  workspace: zero-filled before first use,
 *   left zero-filled, >= usk_linear_batch_workspace_bytes(...). */
USK_API size_t usk_linear_batch_workspace_bytes(const usk_plan* plan, const int32_t* layers,
                                                const int64_t* ranges, int32_t n);
USK_API usk_status usk_linear_batch(const usk_plan* plan, const void* sketch, const int32_t* layers,
                                    const int64_t* ranges, int32_t n, const void* x, int32_t x_dtype,
                                    void* const* y, int32_t y_dtype, void* workspace,
                                    size_t workspace_bytes, usk_stream stream);

/* Prefill form of usk_linear_batch: T tokens through several layers that share one input
 * (q|k|v, gate|up), the paper's decompression -> computation done once per
 * group: the W' rows of all n layers are rebuilt into consecutive rows of `workspace`
 * (usk_reconstruct's bytes), then ONE tcgen05 GEMM over the concatenated rows writes each layer's
 * columns straight into its own y[k].  For k < n, t < T:
 *   y[k][t, o - ranges[2k]] = sum_j x[t, j] * w'_{layers[k]}(o, j),  o in [ranges[2k], ranges[2k+1]).
 *   x: device [T, in] bf16 (bf16 plans); y[k]: device [T, rows_k] of y_dtype, row-major, contiguous.
 *   Same numerics as n calls of usk_linear with T tokens (fp32 accumulation of the same products
 *   in the same K order).  One GEMM needs every layer but the last to have rows_k % 32 == 0 and
 *   full ranges; otherwise the layers run one after another through the same workspace (same
 *   results).  T == 1 is usk_linear_batch.  workspace: >= usk_linear_batch_tokens_workspace_bytes
 *   (...), 16-B aligned.  USK_EUNSUPPORTED for fp32 plans or fp32 x with T > 1. */
USK_API size_t usk_linear_batch_tokens_workspace_bytes(const usk_plan* plan, const int32_t* layers,
                                                       const int64_t* ranges, int32_t n, int64_t T);
USK_API usk_status usk_linear_batch_tokens(const usk_plan* plan, const void* sketch, const int32_t* layers,
                                           const int64_t* ranges, int32_t n, const void* x, int32_t x_dtype,
                                           int64_t T, void* const* y, int32_t y_dtype, void* workspace,
                                           size_t workspace_bytes, usk_stream stream);

/* The computation stage alone ("computation"): Y_k = X . W'_k^T for n weight
 * blocks stored back to back, row-major, in w (bf16 [sum rows_k, in]; e.g. W' rebuilt by
 * usk_reconstruct_batch), ONE tcgen05 GEMM whose epilogue writes block k's columns to y[k]
 * ([T, rows_k] of y_dtype, contiguous).  Lets a caller overlap the decompression of the next group
 * with this group's GEMM (two workspaces, two streams).  rows[k] % 32 == 0 for k < n - 1, n <= 8;
 * x, w 16-B aligned; in % 8 == 0.  Same results as usk_linear_batch_tokens on the same W'. */
USK_API usk_status usk_gemm_tokens(const void* x, int64_t T, int64_t in, const void* w, const int64_t* rows,
                                   int32_t n, void* const* y, int32_t y_dtype, usk_stream stream);

/* Output-sharded decode with the y all-gather fused into the split-K reduction (SURVEY 8(e),
 * north star "each linear's output features are sharded for inference"; B200-native collective in
 * place of an NCCL all-gather).  Rank my_rank of n_peers computes rows [ranges[2k], ranges[2k+1])
 * of each layer as usk_linear_batch does (query-layout plans), but its reduce kernel stores every
 * row at its GLOBAL position o in the full y of EVERY rank (y_peer: device pointers of the peers'
 * buffers mapped into this process -- CUDA IPC / symmetric memory over NVLink), then raises this
 * rank's flag sig_peer[p][my_rank] = *epoch + 1 in every rank's signal array (system-scope release
 * after all of its rows are visible).  usk_peer_wait, enqueued by each rank after its call, waits
 * (acquire) until all n_peers flags of its own signal array reach *epoch + 1 and advances *epoch:
 * then every rank's full y holds every rank's rows.  Graph-replayable (the epoch lives on the device).
 *   peers: host struct; y_peer host array [n_peers * n] (y_peer[p * n + k] = rank p's full y of
 *          layers[k], out_features elements of y_dtype, 16-B aligned); sig_peer host array [n_peers]
 *          of device uint32[n_peers] arrays (zero-filled before first use); epoch: device uint32, the
 *          same value on every rank (0 at first use).
 * The spin of usk_peer_wait is bounded: a peer that never signals is reported by usk_check (USK_ECUDA). */
typedef struct {
  int32_t n_peers;            /* ranks P in [1, 8] */
  int32_t my_rank;
  void* const* y_peer;        /* host [P * n] device pointers */
  uint32_t* const* sig_peer;  /* host [P] device pointers */
  uint32_t* epoch;            /* device uint32 */
} usk_peers;
USK_API usk_status usk_linear_batch_peers(const usk_plan* plan, const void* sketch, const int32_t* layers,
                                          const int64_t* ranges, int32_t n, const void* x, int32_t x_dtype,
                                          int32_t y_dtype, const usk_peers* peers, void* workspace,
                                          size_t workspace_bytes, usk_stream stream);
USK_API usk_status usk_peer_wait(const usk_plan* plan, const usk_peers* peers, usk_stream stream);

/* Aggregated-gradient baseline of finetuning (§3.3, Figure 4a; SPEC.md
 * aggregated_backward): the gradient of a shared sketch state is the sum of the gradients of the
 * weights mapped to it.  For every weight (o, j) of `layer` and every sketch row i,
 *   cell_grad[c_i(o, j) - cell_begin] += grad[o, j],
 * summed in 2^-48 fixed point (q = rint(g * 2^48) as int64, result fl32(fl64(sum) * 2^-48)), so the
 * result does not depend on the summation order (DESIGN.md ledger L26; |sum| < 2^15).
 *   grad: device [out, in] row-major of grad_dtype (USK_F32 / USK_BF16); cell_grad: device
 *   float[n_cells of the layer]; workspace: device, >= usk_aggregate_grad_workspace_bytes, 16-B
 *   aligned, zero-filled before first use -- every call leaves it zero-filled.
 * Raw-state plans only (USK_EUNSUPPORTED for state_bits != 0).  The STE alternative (identity
 * backward through build + reconstruct) needs no kernel of its own. */
USK_API size_t usk_aggregate_grad_workspace_bytes(const usk_plan* plan, int32_t layer);
USK_API usk_status usk_aggregate_grad(const usk_plan* plan, int32_t layer, const void* grad, int32_t grad_dtype,
                                      float* cell_grad, void* workspace, size_t workspace_bytes,
                                      usk_stream stream);

/* Compression report of one layer (SPEC stats; untouched weights PAPER.md:616-619; Table 3
 * unoccupied states), computed on the device from the original weights and the sketch:
 *   counts (device int64[USK_STATS_N]) receives, for the layer's weights w and reconstructions w':
 *   [0] weights, [1] untouched (w' bits == w bits), [2] sign errors (both nonzero, signs differ),
 *   [3] zero weights, [4..10] histogram of r = fl32(fl32(|w - w'|) / |w|) over nonzero w:
 *   r == 0, (0, 1e-3), [1e-3, 1e-2), [1e-2, 0.1), [0.1, 1), [1, 10), [10, inf);
 *   [11] cells of the layer, [12] unoccupied cells (no weight of the layer maps to them).
 *   W: device [out, in] of the plan dtype; workspace: device, >= usk_stats_workspace_bytes,
 *   zero-filled before first use, left zero-filled.  Integer counts: deterministic. */
#define USK_STATS_N 13
USK_API size_t usk_stats_workspace_bytes(const usk_plan* plan, int32_t layer);
USK_API usk_status usk_stats(const usk_plan* plan, const void* sketch, int32_t layer, const void* W, int64_t* counts,
                             void* workspace, size_t workspace_bytes, usk_stream stream);

/* Synchronises `stream`, returns and clears the plan's sticky device error (USK_ENONFINITE),
 * or USK_ECUDA on a CUDA error, else USK_OK. */
USK_API usk_status usk_check(const usk_plan* plan, usk_stream stream);

USK_API void usk_plan_destroy(usk_plan* plan);

USK_API const char* usk_status_string(usk_status status);
USK_API const char* usk_last_error(void);

/* Number of kernel launches this thread issued through the ABI since the last reset
 * (bench evidence for "gpu_launches"). */
USK_API int64_t usk_launch_count(int32_t reset);

/* Tuning-only kernel trace (active only when the environment variable USK_TRACE is set when the
 * library first launches a query kernel).  Every sketch-GEMV / reconstruct launch then writes 4
 * %globaltimer stamps per CTA (start, staged, compute done, exit) into a device ring; launch
 * slots are assigned when the launch is ISSUED, so a captured CUDA graph rewrites the same slots
 * on every replay.  usk_trace_read synchronises the device, copies up to cap_stamps stamps
 * (4 per CTA, launches in issue order) into `stamps` and up to cap_launches grid sizes into
 * `grids` (host buffers) and returns the number of launches recorded (0 when tracing is off).
 * usk_trace_reset forgets all slots (call before capturing a new graph). */
USK_API int32_t usk_trace_read(uint64_t* stamps, int64_t cap_stamps, int32_t* grids, int32_t cap_launches);
USK_API void usk_trace_reset(void);

#ifdef __cplusplus
}
#endif

#endif /* USK_H */
