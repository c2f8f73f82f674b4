/*
 * usk_oracle.c -- plain, slow, obviously-correct CPU ORACLE of the UltraSketchLLM
 * (arXiv 2506.17255) index-free multi-row AbsMaxMin sketch.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code,
 * header, table or constant generator with the CUDA product path
 * (paper_2506_17255_b200/csrc); the two meet only in the written contract
 * ("Allocation").
 *
 * Everything is scalar C99, no intrinsics, compiled -O2 -fno-fast-math
 * -ffp-contract=off.  Values are compared as IEEE doubles (exact for fp32/bf16),
 * never as packed integer keys, so the oracle does not share the GPU's encoding.
 *
 * Citations: PAPER.md:<line> (section / equation), SPEC.md:<line>.
 *
 * Parity status per function (details in DESIGN.md "Oracle pins"):
 *   uo_update / uo_retrieve / uo_sketch_unit / uo_retrieve_unit  -- pinned (SPEC worked
 *       examples, brute-force preimage enumeration, underestimate, order independence)
 *   uo_hash_index  -- exact values are OUR contract (paper fixes only "independent hash
 *       functions"): "parity unpinned" for individual index values;
 *       pinned statistically (Table 3 empty fractions, untouched closed forms).
 *   uo_allocate / uo_plan -- pinned (SPEC allocation examples, conservation, monotonicity,
 *       scale invariance, bpw accounting vs Table 1 arithmetic); class boundaries and the
 *       remainder order are our reading (L9/L10): "parity unpinned" for those.
 *   per-class sketch rows (uo_plan class_rows, uo_allocate Mc, ledger L30) --
 *       pinned (hand-worked allocation, reduction to the uniform plan, conservation, the set-based
 *       enumerator per unit incl. LAYER units, Appendix B's untouched closed form per class).
 *   key-group scores (uo_plan2 score_group = 8 under USK-XG, ledger L33) -- pinned (group means
 *       computed apart in tests/test_oracle_xg_classes.py fed to the pinned allocator; uniform
 *       groups, class order, USK-X plans unchanged, uniform saliency gives identical plans).
 *   output-row units (UO_GRAN_OUTROW, ledger L31) -- pinned (byte-identical to
 *       input-dim units of W^T, set-based enumerator per unit, accounting, untouched closed form).
 *   uo_importance -- pinned (SPEC Eq. 7 examples, constant activations).
 *   uo_linear_rows -- pinned (numpy fp64 matmul of the oracle-verified W').
 *   uo_aggregate_grad (aggregated-gradient baseline) -- pinned (SPEC example
 *       0.1 + -0.3 -> -0.2, the exact fp64 sum within the fixed-point resolution, injective
 *       mapping = identity, central finite differences of a shared-parameter loss).
 *   uo_quantize / uo_dequantize / uo_pack_codes / uo_f32_to_bf16_rne (stacked state
 *       quantisation) -- pinned (SPEC quant worked examples, round-trip error
 *       bound <= scale/2, code range, unoccupied -> 0, torch's bf16 RNE conversion).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* status codes: numerically identical to include/usk.h by written contract only */
#define UO_OK 0
#define UO_EINVAL 1
#define UO_ESHAPE 2
#define UO_EBUDGET 3
#define UO_ENONFINITE 4

#define UO_F32 0
#define UO_BF16 1

#define UO_HASH_X 0
#define UO_HASH_IDENTITY 1
#define UO_HASH_XG 2 /* USK-X with unit keys shared by groups of UO_KEY_GROUP consecutive units (ledger L32) */
#define UO_KEY_GROUP 8

#define UO_GRAN_ROW 0
#define UO_GRAN_LAYER 1
#define UO_GRAN_OUTROW 2 /* one unit per OUTPUT row o of W [out, in], positions p = j (ledger L31) */

/* sketch variants (Appendix C.2) */
#define UO_ABSMAXMIN 0 /* the paper's sketch: keep min |.|, retrieve max |.| */
#define UO_ABSMINMAX 1 /* "changes the order of the min and max operations" */
#define UO_COUNTMIN 2  /* "adding the current weight ... retrieves ... minimum absolute value" */

/* ------------------------------------------------------------------------------------
 * Hash family "USK-X" (paper Eq. 3, PAPER.md:239-243:
 * I = H(Addr(w)) with independent H_0..H_{M-1}; Addr(w) is the natural, storage-free
 * index of the weight inside its compression unit).
 * ------------------------------------------------------------------------------------ */
uint64_t uo_splitmix64(uint64_t x) {
  uint64_t z;
  x = x + 0x9E3779B97F4A7C15ull;
  z = x;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

uint32_t uo_fmix32(uint32_t h) {
  h ^= h >> 16;
  h *= 0x85EBCA6Bu;
  h ^= h >> 13;
  h *= 0xC2B2AE35u;
  h ^= h >> 16;
  return h;
}

/* rho_i: per sketch row position salt */
uint32_t uo_row_salt(uint64_t seed, int32_t row) {
  return (uint32_t)uo_splitmix64(seed + 0x200ull + (uint64_t)row);
}

/* kappa_i: per sketch row key salt */
uint32_t uo_row_key_salt(uint64_t seed, int32_t row) {
  return (uint32_t)uo_splitmix64(seed + 0x300ull + (uint64_t)row);
}

/* K_u: per compression unit u = (layer l, unit t) */
uint32_t uo_unit_key(uint64_t seed, uint32_t layer, uint32_t t) {
  uint64_t lt = ((uint64_t)layer << 32) | (uint64_t)t;
  return (uint32_t)uo_splitmix64(seed ^ uo_splitmix64(lt));
}

/* R_i(p) = fmix32(p ^ rho_i): per position and row, shared by every unit */
uint32_t uo_position_mix(uint64_t seed, int32_t row, uint32_t p) {
  return uo_fmix32(p ^ uo_row_salt(seed, row));
}

/* h_i(u, p) = R_i(p) ^ fmix32(K_u ^ kappa_i) */
uint32_t uo_hash_word(uint64_t seed, uint32_t layer, uint32_t t, int32_t row, uint32_t p) {
  return uo_position_mix(seed, row, p) ^ uo_fmix32(uo_unit_key(seed, layer, t) ^ uo_row_key_salt(seed, row));
}

/* idx_i(u, p) in [0, ncols):
 *   short units (ncols <= 2^16): floor((h mod 2^23) * ncols / 2^23)
 *   long units:                  floor(h * ncols / 2^32) */
uint32_t uo_hash_index(int32_t kind, uint64_t seed, uint32_t layer, uint32_t t, int32_t row,
                       uint32_t p, uint32_t ncols) {
  if (kind == UO_HASH_IDENTITY) return p % ncols; /* SPEC.md:54 test_hash: flat_index mod columns */
  /* USK-XG (DESIGN.md ledger L32): the M hash functions H_i of PAPER.md:243 are shared by the
   * UO_KEY_GROUP consecutive units t = 8g .. 8g+7 of a layer -- the unit key is that of the group,
   * K_(l, floor(t / 8)) -- and unchanged otherwise */
  if (kind == UO_HASH_XG) t = t / UO_KEY_GROUP;
  {
    uint32_t h = uo_hash_word(seed, layer, t, row, p);
    if (ncols <= 65536u) return (uint32_t)(((uint64_t)(h & 0x7FFFFFu) * (uint64_t)ncols) >> 23);
    return (uint32_t)(((uint64_t)h * (uint64_t)ncols) >> 32);
  }
}

/* ------------------------------------------------------------------------------------
 * Cell values.  A cell / weight is held as its raw bit pattern (bf16 in the low 16 bits).
 * ------------------------------------------------------------------------------------ */
static double uo_value(int32_t dtype, uint32_t bits) {
  float f;
  uint32_t b = (dtype == UO_BF16) ? (bits << 16) : bits;
  memcpy(&f, &b, sizeof f);
  return (double)f;
}

static uint32_t uo_inf_bits(int32_t dtype) { return dtype == UO_BF16 ? 0x7F80u : 0x7F800000u; }
static uint32_t uo_load_bits(int32_t dtype, const void* base, int64_t idx) {
  return dtype == UO_BF16 ? (uint32_t)((const uint16_t*)base)[idx] : ((const uint32_t*)base)[idx];
}

/* Eq. 4: S[i,I_i] = (Abs(S[i,I_i]) > Abs(X)) ? X : S[i,I_i].
 * Tie |X| == |S| with opposite signs: prefer the non-negative value (L2,
 * SPEC.md:110).  Returns the new cell. */
uint32_t uo_update(int32_t dtype, uint32_t cell, uint32_t x) {
  double s = uo_value(dtype, cell), v = uo_value(dtype, x);
  if (fabs(s) > fabs(v)) return x;
  if (fabs(s) == fabs(v) && signbit(s) && !signbit(v)) return x;
  return cell;
}

/* Eq. 5: w' = Max_i S[i][H_i(Addr(w))], "Max" read as the maximum
 * absolute value returning the signed cell (L1); tie -> the
 * non-negative value (L2). */
uint32_t uo_retrieve(int32_t dtype, const uint32_t* bonded, int32_t M) {
  uint32_t best = bonded[0];
  int32_t i;
  for (i = 1; i < M; i++) {
    double b = uo_value(dtype, best), c = uo_value(dtype, bonded[i]);
    if (fabs(c) > fabs(b) || (fabs(c) == fabs(b) && signbit(b) && !signbit(c))) best = bonded[i];
  }
  return best;
}

static int uo_finite(int32_t dtype, uint32_t bits) { return isfinite(uo_value(dtype, bits)); }
/* Variants (Appendix C.2; DESIGN.md ledger L27).  AbsMinMax keeps the colliding
 * weight of MAXIMUM |.| (cells start at +0, ties -> non-negative) and retrieves the bonded cell of
 * MINIMUM |.| (ties -> non-negative).  CountMin cells hold the sum of their weights (2^-48 fixed
 * point, as the aggregated gradient, L26, rounded to the weight dtype) and retrieve like AbsMinMax. */
static uint32_t uo_update_absminmax(int32_t dtype, uint32_t cell, uint32_t x) {
  double s = uo_value(dtype, cell), v = uo_value(dtype, x);
  if (fabs(v) > fabs(s)) return x;
  if (fabs(s) == fabs(v) && signbit(s) && !signbit(v)) return x;
  return cell;
}

uint32_t uo_retrieve_v(int32_t variant, int32_t dtype, const uint32_t* bonded, int32_t M) {
  uint32_t best = bonded[0];
  int32_t i;
  if (variant == UO_ABSMAXMIN) return uo_retrieve(dtype, bonded, M);
  for (i = 1; i < M; i++) {
    double b = uo_value(dtype, best), c = uo_value(dtype, bonded[i]);
    if (fabs(c) < fabs(b) || (fabs(c) == fabs(b) && signbit(b) && !signbit(c))) best = bonded[i];
  }
  return best;
}

/* fp32 -> weight dtype bits (bf16: round to nearest even) */
static uint32_t uo_from_float(int32_t dtype, float f) {
  uint32_t b;
  memcpy(&b, &f, 4);
  return dtype == UO_BF16 ? (b + 0x7FFFu + ((b >> 16) & 1u)) >> 16 : b;
}



/* One compression unit ("S in AbsMaxMin is initialized as inf";
 * select Eq. 3, update Eq. 4).  Inserts the n (position, weight) pairs in the order
 * given (any order gives the same state).  cells: M*N, row-major by sketch
 * row. */
int32_t uo_sketch_unit(int32_t dtype, const uint32_t* w_bits, const uint32_t* pos, int64_t n,
                       int32_t hash_kind, uint64_t seed, uint32_t layer, uint32_t t, int32_t M,
                       uint32_t N, uint32_t* cells) {
  int64_t k;
  int32_t i;
  uint32_t c;
  if (M < 1 || N < 1) return UO_EINVAL;
  for (i = 0; i < M; i++)
    for (c = 0; c < N; c++) cells[(int64_t)i * N + c] = uo_inf_bits(dtype);
  for (k = 0; k < n; k++) {
    if (!uo_finite(dtype, w_bits[k])) return UO_ENONFINITE;
    for (i = 0; i < M; i++) {
      uint32_t idx = uo_hash_index(hash_kind, seed, layer, t, i, pos[k], N);
      uint32_t* cell = &cells[(int64_t)i * N + idx];
      *cell = uo_update(dtype, *cell, w_bits[k]);
    }
  }
  return UO_OK;
}

/* one unit under a variant (cells as in uo_sketch_unit) */
int32_t uo_sketch_unit_v(int32_t variant, int32_t dtype, const uint32_t* w_bits, const uint32_t* pos, int64_t n,
                         int32_t hash_kind, uint64_t seed, uint32_t layer, uint32_t t, int32_t M, uint32_t N,
                         uint32_t* cells) {
  int64_t k, c;
  int32_t i;
  int64_t* acc;
  if (variant == UO_ABSMAXMIN) return uo_sketch_unit(dtype, w_bits, pos, n, hash_kind, seed, layer, t, M, N, cells);
  if (M < 1 || N < 1) return UO_EINVAL;
  for (k = 0; k < n; k++)
    if (!uo_finite(dtype, w_bits[k])) return UO_ENONFINITE;
  if (variant == UO_ABSMINMAX) {
    for (c = 0; c < (int64_t)M * N; c++) cells[c] = 0u; /* +0 */
    for (k = 0; k < n; k++)
      for (i = 0; i < M; i++) {
        uint32_t* cell = &cells[(int64_t)i * N + uo_hash_index(hash_kind, seed, layer, t, i, pos[k], N)];
        *cell = uo_update_absminmax(dtype, *cell, w_bits[k]);
      }
    return UO_OK;
  }
  if (variant != UO_COUNTMIN) return UO_EINVAL;
  acc = (int64_t*)calloc((size_t)M * N, sizeof(int64_t));
  for (k = 0; k < n; k++) {
    const int64_t q = llrint(uo_value(dtype, w_bits[k]) * 281474976710656.0); /* 2^48 */
    for (i = 0; i < M; i++) acc[(int64_t)i * N + uo_hash_index(hash_kind, seed, layer, t, i, pos[k], N)] += q;
  }
  for (c = 0; c < (int64_t)M * N; c++)
    cells[c] = uo_from_float(dtype, (float)((double)acc[c] * (1.0 / 281474976710656.0)));
  free(acc);
  return UO_OK;
}

/* Retrieval of n positions from one unit (hash, batched gather,
 * interpret with Max). */
int32_t uo_retrieve_unit(int32_t dtype, const uint32_t* cells, int32_t hash_kind, uint64_t seed,
                         uint32_t layer, uint32_t t, int32_t M, uint32_t N, const uint32_t* pos,
                         int64_t n, uint32_t* out_bits) {
  int64_t k;
  int32_t i;
  uint32_t bonded[8];
  if (M < 1 || M > 8 || N < 1) return UO_EINVAL;
  for (k = 0; k < n; k++) {
    for (i = 0; i < M; i++)
      bonded[i] = cells[(int64_t)i * N + uo_hash_index(hash_kind, seed, layer, t, i, pos[k], N)];
    out_bits[k] = uo_retrieve(dtype, bonded, M);
  }
  return UO_OK;
}

/* ------------------------------------------------------------------------------------
 * Eq. 7: I_j = E[a_j^2] = (1/N) sum_k a_{k,j}^2.  A is [N, d]
 * row-major fp32; sequential fp64 sum over k.
 * ------------------------------------------------------------------------------------ */
int32_t uo_importance(const float* A, int64_t N, int64_t d, double* I) {
  int64_t j, k;
  if (N < 1 || d < 1) return UO_ESHAPE;
  for (j = 0; j < d; j++) {
    double s = 0.0;
    for (k = 0; k < N; k++) {
      double a = (double)A[k * d + j];
      s += a * a;
    }
    I[j] = s / (double)N;
  }
  return UO_OK;
}

/* ------------------------------------------------------------------------------------
 * Allocation (§3.4: "assign I_j / sum_i I_i x Mem(Sketch)"; categories
 * PAPER.md:523-528).  Deterministic integer reading, DESIGN.md "Allocation" (L8-L12):
 *   q_u = floor(s_u / s_max * 2^24); rank by (q desc, u asc); class c = floor(rank*C/U);
 *   W_c = sum_{u in c} q_u L_u; x_c = T W_c / (W n_c M); N_c = max(min_cols, floor x_c)
 *   with water-filling of floor-clamped classes; largest remainder in (frac desc, c asc).
 * ------------------------------------------------------------------------------------ */
typedef unsigned __int128 uo_u128;

typedef struct {
  uint64_t q;
  int64_t u;
} uo_rank_item;

static int uo_rank_cmp(const void* a, const void* b) {
  const uo_rank_item* x = (const uo_rank_item*)a;
  const uo_rank_item* y = (const uo_rank_item*)b;
  if (x->q != y->q) return x->q > y->q ? -1 : 1; /* q descending */
  return x->u < y->u ? -1 : (x->u > y->u ? 1 : 0); /* u ascending */
}

typedef struct {
  uint64_t key;
  int32_t c;
} uo_rem_item;

static int uo_rem_cmp(const void* a, const void* b) {
  const uo_rem_item* x = (const uo_rem_item*)a;
  const uo_rem_item* y = (const uo_rem_item*)b;
  if (x->key != y->key) return x->key > y->key ? -1 : 1;
  return x->c < y->c ? -1 : (x->c > y->c ? 1 : 0);
}

/* s_u: unit scores (>= 0, finite); L_u: unit lengths (weights per unit; pass 1 for a
 * common length); T: cells available; C classes; Mc[c]: sketch rows of class c (ledger L30: the
 * class's share of the cells is split into Mc[c] rows of N_c columns, so x_c = T W_c / (W n_c
 * Mc[c])); min_cols floor.  Outputs: cls[U], ncols[U]. */
int32_t uo_allocate(int64_t U, const double* s_u, const uint64_t* L_u, int64_t T, int32_t C,
                    const int32_t* Mc, int32_t min_cols, uint8_t* cls, int32_t* ncols) {
  int64_t u, r;
  int32_t c;
  double s_max = 0.0;
  uint64_t* q;
  uo_rank_item* items;
  int64_t n_c[256];
  uo_u128 W_c[256];
  int active[256];
  int64_t N_c[256];
  uo_u128 num_c[256], den_c[256];
  if (U < 1) return UO_ESHAPE;
  if (C < 1 || C > 255 || min_cols < 1 || T < 0) return UO_EINVAL;
  for (c = 0; c < C; c++)
    if (Mc[c] < 1 || Mc[c] > 8) return UO_EINVAL;
  q = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)U);
  items = (uo_rank_item*)malloc(sizeof(uo_rank_item) * (size_t)U);
  for (u = 0; u < U; u++) {
    if (!(s_u[u] >= 0.0) || !isfinite(s_u[u])) {
      free(q);
      free(items);
      return UO_EINVAL;
    }
    if (s_u[u] > s_max) s_max = s_u[u];
  }
  /* step 2: fixed point */
  for (u = 0; u < U; u++) q[u] = (s_max > 0.0) ? (uint64_t)floor((s_u[u] / s_max) * 16777216.0) : 1u;
  /* step 3: rank, classes */
  for (u = 0; u < U; u++) {
    items[u].q = q[u];
    items[u].u = u;
  }
  qsort(items, (size_t)U, sizeof(uo_rank_item), uo_rank_cmp);
  for (c = 0; c < C; c++) {
    n_c[c] = 0;
    W_c[c] = 0;
  }
  for (r = 0; r < U; r++) {
    int64_t uu = items[r].u;
    int32_t cc = (int32_t)((r * (int64_t)C) / U);
    cls[uu] = (uint8_t)cc;
    n_c[cc] += 1;
    W_c[cc] += (uo_u128)q[uu] * (uo_u128)L_u[uu];
  }
  /* feasibility of the floor */
  {
    int64_t floor_cells = 0;
    for (c = 0; c < C; c++) floor_cells += n_c[c] * (int64_t)Mc[c] * (int64_t)min_cols;
    if (floor_cells > T) {
      free(q);
      free(items);
      return UO_EBUDGET;
    }
  }
  /* steps 4-5: proportional share with water-filling of clamped classes */
  for (c = 0; c < C; c++) active[c] = n_c[c] > 0;
  for (;;) {
    uo_u128 Wa = 0;
    int64_t Ta = T;
    int changed = 0;
    for (c = 0; c < C; c++) {
      if (n_c[c] == 0) continue;
      if (active[c])
        Wa += W_c[c];
      else
        Ta -= n_c[c] * (int64_t)Mc[c] * (int64_t)min_cols;
    }
    for (c = 0; c < C; c++) {
      if (!active[c]) continue;
      num_c[c] = (uo_u128)Ta * W_c[c];
      den_c[c] = Wa * (uo_u128)n_c[c] * (uo_u128)Mc[c];
      N_c[c] = (den_c[c] == 0) ? 0 : (int64_t)(num_c[c] / den_c[c]);
      if (N_c[c] < min_cols) {
        active[c] = 0;
        changed = 1;
      }
    }
    if (!changed) break;
  }
  for (c = 0; c < C; c++)
    if (!active[c]) N_c[c] = min_cols;
  /* step 6: largest remainder over the unclamped classes */
  {
    int64_t left = T;
    uo_rem_item rem[256];
    int32_t n_rem = 0, k;
    for (c = 0; c < C; c++) left -= n_c[c] * (int64_t)Mc[c] * N_c[c];
    for (c = 0; c < C; c++) {
      if (!active[c]) continue;
      rem[n_rem].key = (uint64_t)(((num_c[c] % den_c[c]) << 32) / den_c[c]);
      rem[n_rem].c = c;
      n_rem++;
    }
    qsort(rem, (size_t)n_rem, sizeof(uo_rem_item), uo_rem_cmp);
    for (k = 0; k < n_rem; k++) {
      int32_t cc = rem[k].c;
      int64_t need = n_c[cc] * (int64_t)Mc[cc];
      if (need <= left) {
        N_c[cc] += 1;
        left -= need;
      }
    }
  }
  for (u = 0; u < U; u++) ncols[u] = (int32_t)N_c[cls[u]];
  free(q);
  free(items);
  return UO_OK;
}

/* ------------------------------------------------------------------------------------
 * Model plan (scopes per PAPER.md:331-334).
 *   ROW:   unit (l, t) = input dims [t*g, (t+1)*g) of layer l (L6/L7); each
 *          layer is one budget scope of floor(bpw * numel_l) bits ("Mem(Sketch) is the target
 *          storage by all sketch states in a layer"), minus the class map
 *          U_l * ceil(log2 C) bits when C > 1.
 *   LAYER: one unit per layer; one scope over the model; unit score = mean row
 *          importance, share proportional to score x numel (L8).
 * Offsets: exclusive prefix sum of M * N_u over units in (layer, t) order.
 * layer_acct[4*l + {0,1,2,3}] = {budget bits, class-map bits, cells T (ROW; -1 for
 * LAYER), achieved bits (states + class map)}.
 * ------------------------------------------------------------------------------------ */
static int32_t uo_ceil_log2(int32_t C) {
  int32_t b = 0;
  while ((1 << b) < C) b++;
  return b;
}

/* Stacked state quantisation (q = 4 or 8 bits per state; PAPER.md:348-350,
 * Table 1 "+ q4"/"+ q8"): states are stored as codes in groups of G consecutive cells of a
 * layer with one fp32 scale per group.  Each layer's cells start at a multiple of G (layers are
 * padded; padding cells are unoccupied), so a layer stores ceil(cells/G) groups of q*G + 32 bits
 * (DESIGN.md ledger L25).  ROW scope: T = floor((budget - meta) / (q*G + 32)) * G; LAYER scope:
 * T = (floor(budget / (q*G + 32)) - n_layers) * G (one partial group per layer). */
static int64_t uo_align_up(int64_t x, int64_t a) { return ((x + a - 1) / a) * a; }

/* Two-level (layer x row) allocation ("Front-end layers are more
 * important ... the degradation extent can serve as an important metric"; DESIGN.md ledger L28):
 * the model's cells T are shared among layers in proportion to q_l * numel_l, q_l the layer
 * importance in 2^24 fixed point (as L8), each layer floored at U_l * M * min_cols cells
 * (water-filled), the leftover cells by largest remainder (frac desc, l asc).  Exact integer
 * arithmetic (u128); T_l out. */
int32_t uo_layer_cells(int32_t L, const double* imp, const int64_t* numel, const int64_t* Ul, int32_t M,
                       int32_t min_cols, int64_t T, int64_t* T_l) {
  int32_t l;
  double smax = 0.0;
  uo_u128 w[256], num[256], den[256];
  int active[256];
  int64_t floor_sum = 0, left;
  uo_rem_item rem[256];
  int32_t n_rem = 0, k;
  if (L < 1 || L > 256) return UO_EINVAL;
  for (l = 0; l < L; l++) {
    if (!(imp[l] >= 0.0) || !isfinite(imp[l])) return UO_EINVAL;
    if (imp[l] > smax) smax = imp[l];
  }
  for (l = 0; l < L; l++) {
    const uint64_t ql = (smax > 0.0) ? (uint64_t)floor((imp[l] / smax) * 16777216.0) : 1u;
    w[l] = (uo_u128)ql * (uo_u128)numel[l];
    floor_sum += Ul[l] * (int64_t)M * (int64_t)min_cols;
    active[l] = 1;
  }
  if (floor_sum > T) return UO_EBUDGET;
  for (;;) {
    uo_u128 Wa = 0;
    int64_t Ta = T;
    int changed = 0;
    for (l = 0; l < L; l++) {
      if (active[l]) Wa += w[l];
      else Ta -= Ul[l] * (int64_t)M * (int64_t)min_cols;
    }
    for (l = 0; l < L; l++) {
      if (!active[l]) continue;
      num[l] = (uo_u128)Ta * w[l];
      den[l] = Wa;
      T_l[l] = (Wa == 0) ? 0 : (int64_t)(num[l] / den[l]);
      if (T_l[l] < Ul[l] * (int64_t)M * (int64_t)min_cols) {
        active[l] = 0;
        changed = 1;
      }
    }
    if (!changed) break;
  }
  left = T;
  for (l = 0; l < L; l++) {
    if (!active[l]) T_l[l] = Ul[l] * (int64_t)M * (int64_t)min_cols;
    left -= T_l[l];
  }
  for (l = 0; l < L; l++) {
    if (!active[l] || den[l] == 0) continue;
    rem[n_rem].key = (uint64_t)(((num[l] % den[l]) << 32) / den[l]);
    rem[n_rem].c = l;
    n_rem++;
  }
  qsort(rem, (size_t)n_rem, sizeof(uo_rem_item), uo_rem_cmp);
  for (k = 0; k < n_rem && left > 0; k++, left--) T_l[rem[k].c] += 1;
  return UO_OK;
}

/* score_group (ledger L33): ROW units score by the mean importance of their group of score_group
 * consecutive units -- the key group under USK-XG (8), so the units of a group share a class and N;
 * 1 = every unit its own score (the plain reading of §3.4) */
int32_t uo_plan2(int32_t n_layers, const int64_t* outf, const int64_t* inf, int32_t dtype,
                 const float* const* sal, double bpw, int32_t M, int32_t gran, int32_t g, int32_t C,
                 int32_t min_cols, int32_t q, int32_t G, const double* layer_imp, int64_t topk,
                 const int32_t* class_rows, int32_t score_group, int64_t* unit_base, uint8_t* cls, int32_t* ncols,
                 uint8_t* nrows, int64_t* offsets, int64_t* layer_acct);

int32_t uo_plan(int32_t n_layers, const int64_t* outf, const int64_t* inf, int32_t dtype,
                const float* const* sal, double bpw, int32_t M, int32_t gran, int32_t g, int32_t C,
                int32_t min_cols, int32_t q, int32_t G, const double* layer_imp, int64_t topk,
                const int32_t* class_rows, int64_t* unit_base, uint8_t* cls, int32_t* ncols, uint8_t* nrows,
                int64_t* offsets, int64_t* layer_acct) {
  return uo_plan2(n_layers, outf, inf, dtype, sal, bpw, M, gran, g, C, min_cols, q, G, layer_imp, topk, class_rows, 1,
                  unit_base, cls, ncols, nrows, offsets, layer_acct);
}

int32_t uo_plan2(int32_t n_layers, const int64_t* outf, const int64_t* inf, int32_t dtype,
                 const float* const* sal, double bpw, int32_t M, int32_t gran, int32_t g, int32_t C,
                 int32_t min_cols, int32_t q, int32_t G, const double* layer_imp, int64_t topk,
                 const int32_t* class_rows, int32_t score_group, int64_t* unit_base, uint8_t* cls, int32_t* ncols,
                 uint8_t* nrows, int64_t* offsets, int64_t* layer_acct) {
  int32_t l, c;
  int64_t U = 0, u;
  int32_t state_bits = (dtype == UO_BF16) ? 16 : 32;
  int64_t two_T[256];
  int32_t Mc[256]; /* rows per class: class_rows (ledger L30), or M for every class */
  if (n_layers < 1 || M < 1 || M > 8 || C < 1 || C > 255 || min_cols < 1) return UO_EINVAL;
  for (c = 0; c < C; c++) {
    Mc[c] = class_rows ? class_rows[c] : M;
    if (Mc[c] < 1 || Mc[c] > 8) return UO_EINVAL;
  }
  if (class_rows && layer_imp) return UO_EINVAL; /* two-level floors assume one row count */
  if (q != 0 && q != 4 && q != 8) return UO_EINVAL;
  if (q != 0 && (G < 32 || (G & (G - 1)) != 0)) return UO_EINVAL; /* power of two >= 32 */
  if (!(bpw > 0.0) || !isfinite(bpw)) return UO_EINVAL;
  if (dtype != UO_F32 && dtype != UO_BF16) return UO_EINVAL;
  if (gran != UO_GRAN_ROW && gran != UO_GRAN_LAYER && gran != UO_GRAN_OUTROW) return UO_EINVAL;
  /* output-row units (L31): every unit of a layer has the same score (the saliency is per input
   * dim, so a row's mean is the layer's mean): one class, one unit per row */
  if (gran == UO_GRAN_OUTROW && (C != 1 || g != 1)) return UO_EINVAL;
  for (l = 0; l < n_layers; l++) {
    if (outf[l] < 1 || inf[l] < 1) return UO_ESHAPE;
    if (outf[l] * inf[l] > 0xFFFFFFFFll) return UO_ESHAPE; /* positions are 32-bit */
    if (gran == UO_GRAN_ROW && (g < 1 || inf[l] % g != 0)) return UO_EINVAL;
  }
  /* units */
  for (l = 0; l < n_layers; l++) {
    unit_base[l] = U;
    U += (gran == UO_GRAN_ROW) ? inf[l] / g : (gran == UO_GRAN_OUTROW) ? outf[l] : 1;
  }
  unit_base[n_layers] = U;

  if (topk < 0 || (topk > 0 && (gran == UO_GRAN_LAYER || q != 0))) return UO_EINVAL;
  if (layer_imp) {
    /* two-level: one model budget, split over layers first (raw states, ROW units) */
    int64_t numel_l[256], Ul_l[256], budget = 0, meta_sum = 0, numel_all = 0;
    int32_t st;
    if (gran == UO_GRAN_LAYER || q != 0 || n_layers > 256) return UO_EINVAL;
    for (l = 0; l < n_layers; l++) {
      numel_l[l] = outf[l] * inf[l];
      Ul_l[l] = (gran == UO_GRAN_OUTROW) ? outf[l] : inf[l] / g;
      numel_all += numel_l[l];
      meta_sum += (C > 1) ? Ul_l[l] * (int64_t)uo_ceil_log2(C) : 0;
    }
    budget = (int64_t)floor(bpw * (double)numel_all);
    if (budget < meta_sum) return UO_EBUDGET;
    st = uo_layer_cells(n_layers, layer_imp, numel_l, Ul_l, M, min_cols, (budget - meta_sum) / state_bits, two_T);
    if (st != UO_OK) return st;
  }

  if (gran != UO_GRAN_LAYER) {
    for (l = 0; l < n_layers; l++) {
      int64_t Ul = (gran == UO_GRAN_OUTROW) ? outf[l] : inf[l] / g, t, j;
      int64_t numel = outf[l] * inf[l];
      int64_t budget = (int64_t)floor(bpw * (double)numel);
      int64_t meta = (C > 1) ? Ul * (int64_t)uo_ceil_log2(C) : 0;
      int64_t T;
      double* s_u;
      uint64_t* L_u;
      int32_t st;
      int64_t achieved = meta;
      /* Top-K outliers (App. A): K = min(topk, numel) weights of the layer stored apart as
       * (32-bit flat index, state) pairs, charged to the layer (ledger L29) */
      const int64_t K = topk < numel ? topk : numel;
      const int64_t side = K * (32 + (int64_t)state_bits);
      if (layer_imp) budget = two_T[l] * state_bits + meta; /* the layer's share of the model budget */
      if (budget < meta + side) return UO_EBUDGET;
      achieved += side;
      T = (q == 0) ? (budget - meta - side) / state_bits
                   : ((budget - meta - side) / ((int64_t)q * G + 32)) * G;
      s_u = (double*)malloc(sizeof(double) * (size_t)Ul);
      L_u = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)Ul);
      for (t = 0; t < Ul; t++) {
        double s = 0.0;
        const int64_t sg = (gran == UO_GRAN_ROW && score_group > 1) ? score_group : 1; /* ledger L33 */
        const int64_t t0 = t / sg * sg, t1 = (t0 + sg < Ul) ? t0 + sg : Ul;
        const int64_t ja = (gran == UO_GRAN_OUTROW) ? 0 : t0 * g, jb = (gran == UO_GRAN_OUTROW) ? inf[l] : t1 * g;
        for (j = ja; j < jb; j++) {
          double v = sal && sal[l] ? (double)sal[l][j] : 1.0;
          if (!(v >= 0.0) || !isfinite(v)) {
            free(s_u);
            free(L_u);
            return UO_EINVAL;
          }
          s += v;
        }
        s_u[t] = s / (double)(jb - ja);
        L_u[t] = 1; /* common unit length within a layer */
      }
      st = uo_allocate(Ul, s_u, L_u, T, C, Mc, min_cols, cls + unit_base[l], ncols + unit_base[l]);
      free(s_u);
      free(L_u);
      if (st != UO_OK) return st;
      {
        int64_t cells = 0;
        for (t = 0; t < Ul; t++) cells += (int64_t)Mc[cls[unit_base[l] + t]] * ncols[unit_base[l] + t];
        achieved += (q == 0) ? cells * state_bits : ((cells + G - 1) / G) * ((int64_t)q * G + 32);
      }
      layer_acct[4 * l + 0] = budget;
      layer_acct[4 * l + 1] = meta;
      layer_acct[4 * l + 2] = T;
      layer_acct[4 * l + 3] = achieved;
    }
  } else {
    int64_t numel = 0, budget, T;
    double* s_u = (double*)malloc(sizeof(double) * (size_t)n_layers);
    uint64_t* L_u = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)n_layers);
    int32_t st;
    for (l = 0; l < n_layers; l++) {
      int64_t j;
      double s = 0.0;
      for (j = 0; j < inf[l]; j++) {
        double v = sal && sal[l] ? (double)sal[l][j] : 1.0;
        if (!(v >= 0.0) || !isfinite(v)) {
          free(s_u);
          free(L_u);
          return UO_EINVAL;
        }
        s += v;
      }
      s_u[l] = s / (double)inf[l];
      L_u[l] = (uint64_t)(outf[l] * inf[l]);
      numel += outf[l] * inf[l];
    }
    budget = (int64_t)floor(bpw * (double)numel);
    if (q == 0) {
      T = budget / state_bits;
    } else {
      int64_t ng = budget / ((int64_t)q * G + 32) - n_layers;
      T = (ng > 0 ? ng : 0) * G;
    }
    st = uo_allocate(n_layers, s_u, L_u, T, C, Mc, min_cols, cls, ncols);
    free(s_u);
    free(L_u);
    if (st != UO_OK) return st;
    for (l = 0; l < n_layers; l++) {
      layer_acct[4 * l + 0] = (l == 0) ? budget : 0;
      layer_acct[4 * l + 1] = 0;
      layer_acct[4 * l + 2] = (l == 0) ? T : 0;
      layer_acct[4 * l + 3] = (q == 0) ? (int64_t)Mc[cls[l]] * ncols[l] * state_bits
                                       : (((int64_t)Mc[cls[l]] * ncols[l] + G - 1) / G) * ((int64_t)q * G + 32);
    }
  }
  /* offsets: exclusive prefix sum of M_u * N_u in (layer, t) order (M_u = the rows of the unit's
   * class); with q, each layer starts at a multiple of G */
  for (u = 0; u < U; u++) nrows[u] = (uint8_t)Mc[cls[u]];
  offsets[0] = 0;
  for (l = 0; l < n_layers; l++) {
    if (q != 0) offsets[unit_base[l]] = uo_align_up(offsets[unit_base[l]], G);
    for (u = unit_base[l]; u < unit_base[l + 1]; u++) offsets[u + 1] = offsets[u] + (int64_t)nrows[u] * ncols[u];
  }
  return UO_OK;
}

/* ------------------------------------------------------------------------------------
 * Stacked state quantisation, per group of G cells (SPEC.md quant module: "scale = max|value|
 * over occupied cells of g divided by the max code magnitude (127 for 8-bit, 7 for 4-bit);
 * codes = round(value/scale) clamped; unoccupied cells coded 0; all-zero groups get scale 0";
 * rounding half away from zero, SPEC "DESIGN DECISIONS").  Arithmetic in fp32 (the scale is
 * stored as fp32; DESIGN.md ledger L25): scale = fl32(absmax / qmax), code = roundf(fl32(v /
 * scale)) clamped to [-qmax, qmax].  A cell is occupied iff its raw state is finite (empty
 * cells hold +Inf).  raw: n cells (n a multiple of G) of the dtype; codes: one
 * int8 per cell (unpacked); scales: n / G floats.
 * ------------------------------------------------------------------------------------ */
int32_t uo_quantize(int32_t dtype, const void* raw, int64_t n, int32_t q, int32_t G, int8_t* codes,
                    float* scales) {
  int64_t gi, c;
  const float qmax = (q == 4) ? 7.0f : 127.0f;
  if ((q != 4 && q != 8) || G < 1 || n % G != 0) return UO_EINVAL;
  for (gi = 0; gi < n / G; gi++) {
    float absmax = 0.0f, scale;
    for (c = gi * G; c < (gi + 1) * G; c++) {
      const float v = (float)uo_value(dtype, uo_load_bits(dtype, raw, c));
      if (isfinite(v) && fabsf(v) > absmax) absmax = fabsf(v);
    }
    scale = absmax / qmax;
    scales[gi] = scale;
    for (c = gi * G; c < (gi + 1) * G; c++) {
      const float v = (float)uo_value(dtype, uo_load_bits(dtype, raw, c));
      float r = 0.0f;
      if (isfinite(v) && scale > 0.0f) {
        r = roundf(v / scale);
        if (r > qmax) r = qmax;
        if (r < -qmax) r = -qmax;
      }
      codes[c] = (int8_t)r;
    }
  }
  return UO_OK;
}

/* value = fl32(code * scale) (SPEC.md quant module "value = code x group scale"), returned as
 * fp32 bit patterns: the quantised sketch is then an fp32 sketch for retrieval (Eq. 5). */
int32_t uo_dequantize(int32_t G, const int8_t* codes, const float* scales, int64_t n, uint32_t* f32_bits) {
  int64_t c;
  if (G < 1) return UO_EINVAL;
  for (c = 0; c < n; c++) {
    const float v = (float)codes[c] * scales[c / G];
    memcpy(&f32_bits[c], &v, 4);
  }
  return UO_OK;
}

/* storage of the codes: q = 8 -> one byte (two's complement) per cell; q = 4 -> two cells per
 * byte, the even cell in the low nibble (SPEC "4-bit codes packed two per byte, little-end
 * nibble first"). */
int32_t uo_pack_codes(int32_t q, const int8_t* codes, int64_t n, uint8_t* out) {
  int64_t c;
  if (q == 8) {
    for (c = 0; c < n; c++) out[c] = (uint8_t)codes[c];
  } else if (q == 4) {
    if (n % 2) return UO_EINVAL;
    for (c = 0; c < n / 2; c++)
      out[c] = (uint8_t)(((uint8_t)codes[2 * c] & 0xFu) | (((uint8_t)codes[2 * c + 1] & 0xFu) << 4));
  } else {
    return UO_EINVAL;
  }
  return UO_OK;
}

/* fp32 -> bf16, round to nearest even (finite values): the reconstruction of a quantised bf16
 * plan (the dequantised fp32 value rounded to the weight dtype). */
uint32_t uo_f32_to_bf16_rne(uint32_t b) { return (b + 0x7FFFu + ((b >> 16) & 1u)) >> 16; }

/* ------------------------------------------------------------------------------------
 * Layer-level build / reconstruct / linear over a unit range of one layer.
 * W: [out, in] row-major raw bits (uint16 bf16 or uint32 fp32).  Unit (l, t):
 *   ROW g:  weights (o, j), j in [t g, (t+1) g), position p = (j - t g) * out + o
 *   LAYER:  all weights, position p = j * out + o
 * ncols/offsets: the layer's slice of the plan (offsets relative to the sketch base,
 * in cells).  sketch: raw bits, one cell per element of the dtype.
 * ------------------------------------------------------------------------------------ */
static uint32_t uo_load(int32_t dtype, const void* base, int64_t idx) {
  return dtype == UO_BF16 ? (uint32_t)((const uint16_t*)base)[idx] : ((const uint32_t*)base)[idx];
}
static void uo_store(int32_t dtype, void* base, int64_t idx, uint32_t bits) {
  if (dtype == UO_BF16)
    ((uint16_t*)base)[idx] = (uint16_t)bits;
  else
    ((uint32_t*)base)[idx] = bits;
}

/* The weights (o, j) of unit t: o in [o0, o1), j in [j0, j1) (ledgers L6/L31). */
static void uo_unit_span(int32_t gran, int32_t g, int64_t out, int64_t in, int64_t t, int64_t* o0, int64_t* o1,
                         int64_t* j0, int64_t* j1) {
  *o0 = 0;
  *o1 = out;
  *j0 = 0;
  *j1 = in;
  if (gran == UO_GRAN_ROW) {
    *j0 = t * g;
    *j1 = (t + 1) * g;
  } else if (gran == UO_GRAN_OUTROW) {
    *o0 = t;
    *o1 = t + 1;
  }
}

/* position p of weight (o, j) inside its unit t (the hash input, Eq. 3 "Addr(w)"):
 * ROW: (j - t g) out + o;  LAYER: j out + o;  OUTROW: j */
static uint32_t uo_unit_pos(int32_t gran, int32_t g, int64_t out, int64_t t, int64_t o, int64_t j) {
  if (gran == UO_GRAN_OUTROW) return (uint32_t)j;
  if (gran == UO_GRAN_ROW) return (uint32_t)((j - t * g) * out + o);
  return (uint32_t)(j * out + o);
}

static int64_t uo_unit_of(int32_t gran, int32_t g, int64_t o, int64_t j) {
  return gran == UO_GRAN_ROW ? j / g : gran == UO_GRAN_OUTROW ? o : 0;
}

int32_t uo_build_units(int32_t dtype, const void* W, int64_t out, int64_t in, int32_t layer,
                       int32_t gran, int32_t g, int64_t t_begin, int64_t t_end,
                       const int32_t* ncols, const int64_t* offsets, const uint8_t* nrows, int32_t hash_kind,
                       uint64_t seed, void* sketch, int32_t variant, const uint8_t* exclude) {
  int64_t t;
  for (t = t_begin; t < t_end; t++) {
    const int32_t M = nrows[t]; /* the unit's sketch rows (its class's, ledger L30) */
    int64_t o0, o1, j0, j1, j, o, n, k = 0;
    uint32_t *wb, *pos, *cells;
    int32_t st;
    int64_t c;
    uo_unit_span(gran, g, out, in, t, &o0, &o1, &j0, &j1);
    n = (j1 - j0) * (o1 - o0);
    wb = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)n);
    pos = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)n);
    cells = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)M * (size_t)ncols[t]);
    for (o = o0; o < o1; o++) /* stream W in its row-major order */
      for (j = j0; j < j1; j++) {
        if (exclude && exclude[o * in + j]) continue; /* Top-K outliers are stored apart */
        wb[k] = uo_load(dtype, W, o * in + j);
        pos[k] = uo_unit_pos(gran, g, out, t, o, j);
        k++;
      }
    st = uo_sketch_unit_v(variant, dtype, wb, pos, k, hash_kind, seed, (uint32_t)layer, (uint32_t)t, M,
                          (uint32_t)ncols[t], cells);
    /* Top-K plans (ledger L29): a cell that no remaining (non-outlier) weight maps to holds +0, not
     * the +Inf sentinel.  No non-outlier weight ever retrieves it (each of its bonded cells holds
     * at least its own weight), the reconstruction overlays the outliers, and the GEMV's outlier
     * correction x (w - w'_sketch) then reads a finite w'_sketch (+Inf would give Inf - Inf). */
    if (st == UO_OK && exclude)
      for (c = 0; c < (int64_t)M * ncols[t]; c++)
        if (cells[c] == uo_inf_bits(dtype)) cells[c] = 0u;
    if (st == UO_OK)
      for (c = 0; c < (int64_t)M * ncols[t]; c++) uo_store(dtype, sketch, offsets[t] + c, cells[c]);
    free(wb);
    free(pos);
    free(cells);
    if (st != UO_OK) return st;
  }
  return UO_OK;
}

static uint32_t uo_weight_at(int32_t dtype, const void* sketch, int64_t out, int64_t in,
                             int32_t layer, int32_t gran, int32_t g, const int32_t* ncols,
                             const int64_t* offsets, const uint8_t* nrows, int32_t hash_kind, uint64_t seed,
                             int64_t o, int64_t j, int32_t variant) {
  int64_t t = uo_unit_of(gran, g, o, j);
  const int32_t M = nrows[t];
  uint32_t p = uo_unit_pos(gran, g, out, t, o, j);
  uint32_t N = (uint32_t)ncols[t];
  uint32_t bonded[8];
  int32_t i;
  (void)in;
  for (i = 0; i < M; i++)
    bonded[i] = uo_load(dtype, sketch,
                        offsets[t] + (int64_t)i * N +
                            uo_hash_index(hash_kind, seed, (uint32_t)layer, (uint32_t)t, i, p, N));
  return uo_retrieve_v(variant, dtype, bonded, M);
}

/* W'[o, j] for o in [o_begin, o_end), all j; w_out is [(o_end-o_begin), in] raw bits. */
int32_t uo_reconstruct_rows(int32_t dtype, const void* sketch, int64_t out, int64_t in,
                            int32_t layer, int32_t gran, int32_t g, const int32_t* ncols,
                            const int64_t* offsets, const uint8_t* nrows, int32_t hash_kind, uint64_t seed,
                            int64_t o_begin, int64_t o_end, void* w_out, int32_t variant) {
  int64_t o, j;
  if (o_begin < 0 || o_end > out || o_begin > o_end) return UO_ESHAPE;
  for (o = o_begin; o < o_end; o++)
    for (j = 0; j < in; j++)
      uo_store(dtype, w_out, (o - o_begin) * in + j,
               uo_weight_at(dtype, sketch, out, in, layer, gran, g, ncols, offsets, nrows, hash_kind,
                            seed, o, j, variant));
  return UO_OK;
}

/* W'[o, j] for an explicit list of (o, j) pairs (sampled parity at full size). */
int32_t uo_reconstruct_entries(int32_t dtype, const void* sketch, int64_t out, int64_t in,
                               int32_t layer, int32_t gran, int32_t g, const int32_t* ncols,
                               const int64_t* offsets, const uint8_t* nrows, int32_t hash_kind, uint64_t seed,
                               const int64_t* oj, int64_t n, uint32_t* out_bits, int32_t variant) {
  int64_t k;
  for (k = 0; k < n; k++)
    out_bits[k] = uo_weight_at(dtype, sketch, out, in, layer, gran, g, ncols, offsets, nrows, hash_kind,
                               seed, oj[2 * k], oj[2 * k + 1], variant);
  return UO_OK;
}

/* Linear ("computation stage follows the original inference step"):
 * y[tok, o] = sum_j x[tok, j] * w'(o, j) in fp64, o in [o_begin, o_end).
 * x: [T, in] doubles; y: [T, o_end - o_begin]. */
int32_t uo_linear_rows(int32_t dtype, const void* sketch, int64_t out, int64_t in, int32_t layer,
                       int32_t gran, int32_t g, const int32_t* ncols, const int64_t* offsets,
                       const uint8_t* nrows, int32_t hash_kind, uint64_t seed, const double* x, int64_t T,
                       int64_t o_begin, int64_t o_end, double* y, int32_t variant) {
  int64_t o, j, tok;
  double* wrow;
  if (o_begin < 0 || o_end > out || o_begin > o_end) return UO_ESHAPE;
  wrow = (double*)malloc(sizeof(double) * (size_t)in);
  for (o = o_begin; o < o_end; o++) {
    for (j = 0; j < in; j++)
      wrow[j] = uo_value(dtype, uo_weight_at(dtype, sketch, out, in, layer, gran, g, ncols, offsets,
                                             nrows, hash_kind, seed, o, j, variant));
    for (tok = 0; tok < T; tok++) {
      double s = 0.0;
      for (j = 0; j < in; j++) s += x[tok * in + j] * wrow[j];
      y[tok * (o_end - o_begin) + (o - o_begin)] = s;
    }
  }
  free(wrow);
  return UO_OK;
}

/* Aggregated-gradient baseline ("estimate the gradient of trainable parameters by
 * aggregating gradients from corresponding original weights", Figure 4a; SPEC aggregated_backward:
 * shared_grad[s] = sum of the member gradients mapped to s).  Every weight (o, j) adds its
 * gradient g to the cell (u, i, idx_i(u, p)) of each sketch row i.  The sum is defined in 2^-48
 * fixed point so that it does not depend on the summation order (DESIGN.md ledger L26):
 *   q(g) = rint(g * 2^48) (int64, ties to even), S = sum q (int64), cell_grad = fl32(fl64(S) * 2^-48).
 * grad: [out, in] doubles (exact values of the fp32 / bf16 gradient); cell_grad: the layer's
 * cells (offsets relative to offsets[0]). */
int32_t uo_aggregate_grad(const double* grad, int64_t out, int64_t in, int32_t layer, int32_t gran,
                          int32_t g, int64_t n_units, const int32_t* ncols, const int64_t* offsets,
                          const uint8_t* nrows, int32_t hash_kind, uint64_t seed, float* cell_grad) {
  int64_t t, o, j, c;
  const int64_t n_cells = offsets[n_units] - offsets[0];
  int64_t* acc = (int64_t*)calloc((size_t)(n_cells > 0 ? n_cells : 1), sizeof(int64_t));
  for (t = 0; t < n_units; t++) {
    int64_t o0, o1, j0, j1;
    uo_unit_span(gran, g, out, in, t, &o0, &o1, &j0, &j1);
    for (o = o0; o < o1; o++)
      for (j = j0; j < j1; j++) {
        const uint32_t p = uo_unit_pos(gran, g, out, t, o, j);
        const int64_t q = llrint(grad[o * in + j] * 281474976710656.0); /* 2^48 */
        int32_t i;
        for (i = 0; i < nrows[t]; i++) {
          const uint32_t idx = uo_hash_index(hash_kind, seed, (uint32_t)layer, (uint32_t)t, i, p, (uint32_t)ncols[t]);
          acc[offsets[t] - offsets[0] + (int64_t)i * ncols[t] + idx] += q;
        }
      }
  }
  for (c = 0; c < n_cells; c++) cell_grad[c] = (float)((double)acc[c] * (1.0 / 281474976710656.0));
  free(acc);
  return UO_OK;
}

/* Compression report (SPEC stats: "relative error per element = |w - w'| / |w| (w = 0 counted
 * separately); sign error when sign(w') != sign(w) and both nonzero"; untouched = bit-exact
 * preservation, Table 3 unoccupied states).  counts (int64[13]):
 *   0 weights, 1 untouched (w' bits == w bits), 2 sign errors, 3 zero weights (w == 0),
 *   4..10 relative-error histogram of the nonzero weights, r = fl32(fl32(|w - w'|) / |w|) in fp32
 *   (DESIGN.md ledger L27): [r == 0], (0, 1e-3), [1e-3, 1e-2), [1e-2, 0.1), [0.1, 1), [1, 10),
 *   [10, inf); 11 cells of the layer, 12 unoccupied cells (no weight maps to them).
 * W, Wp: [out, in] raw bits of the weight dtype (Wp = the reconstruction). */
int32_t uo_stats(int32_t dtype, const void* W, const void* Wp, int64_t out, int64_t in, int32_t layer,
                 int32_t gran, int32_t g, int64_t n_units, const int32_t* ncols, const int64_t* offsets,
                 const uint8_t* nrows, int32_t hash_kind, uint64_t seed, int64_t* counts) {
  static const float edges[5] = {1e-3f, 1e-2f, 1e-1f, 1.0f, 10.0f};
  int64_t e, t, o, j, c;
  const int64_t n_cells = offsets[n_units] - offsets[0];
  int32_t* occ = (int32_t*)calloc((size_t)(n_cells > 0 ? n_cells : 1), sizeof(int32_t));
  for (c = 0; c < 13; c++) counts[c] = 0;
  for (e = 0; e < out * in; e++) {
    const uint32_t wb = uo_load_bits(dtype, W, e), pb = uo_load_bits(dtype, Wp, e);
    const float w = (float)uo_value(dtype, wb), wp = (float)uo_value(dtype, pb);
    counts[0]++;
    if (wb == pb) counts[1]++;
    if (w != 0.0f && wp != 0.0f && (signbit(w) != 0) != (signbit(wp) != 0)) counts[2]++;
    if (w == 0.0f) {
      counts[3]++;
    } else {
      const float d = fabsf(w - wp);
      const float r = d / fabsf(w);
      int b = 0;
      if (r > 0.0f) {
        b = 1;
        while (b <= 5 && r >= edges[b - 1]) b++;
      }
      counts[4 + b]++;
    }
  }
  for (t = 0; t < n_units; t++) {
    int64_t o0, o1, j0, j1;
    uo_unit_span(gran, g, out, in, t, &o0, &o1, &j0, &j1);
    for (o = o0; o < o1; o++)
      for (j = j0; j < j1; j++) {
        const uint32_t p = uo_unit_pos(gran, g, out, t, o, j);
        int32_t i;
        for (i = 0; i < nrows[t]; i++)
          occ[offsets[t] - offsets[0] + (int64_t)i * ncols[t] +
              uo_hash_index(hash_kind, seed, (uint32_t)layer, (uint32_t)t, i, p, (uint32_t)ncols[t])]++;
      }
  }
  counts[11] = n_cells;
  for (c = 0; c < n_cells; c++) counts[12] += occ[c] == 0;
  free(occ);
  return UO_OK;
}

/* Top-K outliers (Appendix A: "considers weights with top-k large absolute
 * values as important ones, stores them independently, and keeps their value untouched"):
 * the K weights of largest |w| (ties -> smaller flat index o*in + j), returned as flat indices in
 * ascending order with their raw bits.  Plain selection: K passes over the weights. */
int32_t uo_topk(int32_t dtype, const void* W, int64_t n, int64_t K, int64_t* idx, uint32_t* vals) {
  uint8_t* taken;
  int64_t k, e, c = 0;
  if (K < 0 || K > n) return UO_EINVAL;
  taken = (uint8_t*)calloc((size_t)(n > 0 ? n : 1), 1);
  for (k = 0; k < K; k++) {
    int64_t best = -1;
    double bv = -1.0;
    for (e = 0; e < n; e++) {
      double a;
      if (taken[e]) continue;
      a = fabs(uo_value(dtype, uo_load_bits(dtype, W, e)));
      if (a > bv) {
        bv = a;
        best = e;
      }
    }
    if (best < 0) break; /* only non-finite weights left (the build rejects them) */
    taken[best] = 1;
  }
  for (e = 0; e < n; e++)
    if (taken[e]) {
      idx[c] = e;
      vals[c] = uo_load_bits(dtype, W, e);
      c++;
    }
  free(taken);
  return UO_OK;
}

/* Peak memory model: sum_i Mem(Sketch_i) + max_i Mem(Layer_i). */
int64_t uo_peak_memory(const int64_t* layer_bytes, const int64_t* sketch_bytes, int32_t n) {
  int64_t s = 0, mx = 0;
  int32_t i;
  for (i = 0; i < n; i++) {
    s += sketch_bytes[i];
    if (layer_bytes[i] > mx) mx = layer_bytes[i];
  }
  return s + mx;
}
