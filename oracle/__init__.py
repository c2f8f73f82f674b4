"""CPU oracle of the UltraSketchLLM AbsMaxMin sketch (arXiv 2506.17255).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  It shares no code with
the CUDA product path (``paper_2506_17255_b200``); neither imports the other.

The arithmetic lives in ``usk_oracle.c`` (plain C99, scalar, fp64 references); this module
only marshals numpy arrays through ctypes.  ``brute.py`` is a second, set-based enumerator
of the same definitions for tiny inputs.
"""
from __future__ import annotations

import ctypes as ct
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "usk_oracle.c")
LIB = os.path.join(HERE, "liboracle.so")

F32, BF16 = 0, 1
ABSMAXMIN, ABSMINMAX, COUNTMIN = 0, 1, 2
HASH_X, HASH_IDENTITY, HASH_XG = 0, 1, 2
KEY_GROUP = 8  # USK-XG: units t = 8g..8g+7 of a layer share the unit key K_(l, g) (L32)
GRAN_ROW, GRAN_LAYER, GRAN_OUTROW = 0, 1, 2
OK, EINVAL, ESHAPE, EBUDGET, ENONFINITE = 0, 1, 2, 3, 4


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (no fast-math, no FP contraction)."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        tmp = f"{LIB}.{os.getpid()}.tmp"  # concurrent builders (pytest -n) each rename atomically
        subprocess.check_call(
            ["gcc", "-std=c99", "-O2", "-fno-fast-math", "-ffp-contract=off", "-fPIC", "-shared",
             "-Wall", "-o", tmp, SRC, "-lm"])
        os.replace(tmp, LIB)
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ct.CDLL(build())
        L = _lib
        u32, u64, i32, i64, p = ct.c_uint32, ct.c_uint64, ct.c_int32, ct.c_int64, ct.c_void_p
        L.uo_splitmix64.restype = u64
        L.uo_splitmix64.argtypes = [u64]
        L.uo_fmix32.restype = u32
        L.uo_fmix32.argtypes = [u32]
        L.uo_row_salt.restype = u32
        L.uo_row_salt.argtypes = [u64, i32]
        L.uo_row_key_salt.restype = u32
        L.uo_row_key_salt.argtypes = [u64, i32]
        L.uo_hash_word.restype = u32
        L.uo_hash_word.argtypes = [u64, u32, u32, i32, u32]
        L.uo_unit_key.restype = u32
        L.uo_unit_key.argtypes = [u64, u32, u32]
        L.uo_position_mix.restype = u32
        L.uo_position_mix.argtypes = [u64, i32, u32]
        L.uo_hash_index.restype = u32
        L.uo_hash_index.argtypes = [i32, u64, u32, u32, i32, u32, u32]
        L.uo_update.restype = u32
        L.uo_update.argtypes = [i32, u32, u32]
        L.uo_retrieve.restype = u32
        L.uo_retrieve.argtypes = [i32, p, i32]
        L.uo_sketch_unit.restype = i32
        L.uo_sketch_unit.argtypes = [i32, p, p, i64, i32, u64, u32, u32, i32, u32, p]
        L.uo_retrieve_unit.restype = i32
        L.uo_retrieve_unit.argtypes = [i32, p, i32, u64, u32, u32, i32, u32, p, i64, p]
        L.uo_importance.restype = i32
        L.uo_importance.argtypes = [p, i64, i64, p]
        L.uo_allocate.restype = i32
        L.uo_allocate.argtypes = [i64, p, p, i64, i32, p, i32, p, p]
        L.uo_plan.restype = i32
        L.uo_plan.argtypes = [i32, p, p, i32, p, ct.c_double, i32, i32, i32, i32, i32, i32, i32, p, i64, p, p, p, p, p, p, p]
        L.uo_plan2.restype = i32
        L.uo_plan2.argtypes = [i32, p, p, i32, p, ct.c_double, i32, i32, i32, i32, i32, i32, i32, p, i64, p, i32, p, p, p,
                               p, p, p]
        L.uo_topk.restype = i32
        L.uo_topk.argtypes = [i32, p, i64, i64, p, p]
        L.uo_layer_cells.restype = i32
        L.uo_layer_cells.argtypes = [i32, p, p, p, i32, i32, i64, p]
        L.uo_quantize.restype = i32
        L.uo_quantize.argtypes = [i32, p, i64, i32, i32, p, p]
        L.uo_dequantize.restype = i32
        L.uo_dequantize.argtypes = [i32, p, p, i64, p]
        L.uo_pack_codes.restype = i32
        L.uo_pack_codes.argtypes = [i32, p, i64, p]
        L.uo_aggregate_grad.restype = i32
        L.uo_aggregate_grad.argtypes = [p, i64, i64, i32, i32, i32, i64, p, p, p, i32, u64, p]
        L.uo_f32_to_bf16_rne.restype = u32
        L.uo_f32_to_bf16_rne.argtypes = [u32]
        L.uo_build_units.restype = i32
        L.uo_build_units.argtypes = [i32, p, i64, i64, i32, i32, i32, i64, i64, p, p, p, i32, u64, p, i32, p]
        L.uo_reconstruct_rows.restype = i32
        L.uo_reconstruct_rows.argtypes = [i32, p, i64, i64, i32, i32, i32, p, p, p, i32, u64, i64, i64, p, i32]
        L.uo_reconstruct_entries.restype = i32
        L.uo_reconstruct_entries.argtypes = [i32, p, i64, i64, i32, i32, i32, p, p, p, i32, u64, p, i64, p, i32]
        L.uo_linear_rows.restype = i32
        L.uo_linear_rows.argtypes = [i32, p, i64, i64, i32, i32, i32, p, p, p, i32, u64, p, i64, i64, i64, p, i32]
        L.uo_retrieve_v.restype = u32
        L.uo_retrieve_v.argtypes = [i32, i32, p, i32]
        L.uo_sketch_unit_v.restype = i32
        L.uo_sketch_unit_v.argtypes = [i32, i32, p, p, i64, i32, u64, u32, u32, i32, u32, p]
        L.uo_stats.restype = i32
        L.uo_stats.argtypes = [i32, p, p, i64, i64, i32, i32, i32, i64, p, p, p, i32, u64, p]
        L.uo_peak_memory.restype = i64
        L.uo_peak_memory.argtypes = [p, p, i32]
    return _lib


def _ptr(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(ct.c_void_p)


class OracleError(RuntimeError):
    def __init__(self, status: int, what: str):
        super().__init__(f"{what}: oracle status {status}")
        self.status = status


def _check(st: int, what: str):
    if st != OK:
        raise OracleError(st, what)


# ------------------------------------------------------------------ dtype helpers
def bits_of(w: np.ndarray, dtype: int) -> np.ndarray:
    """Raw bit patterns as uint32 (bf16 in the low 16 bits)."""
    if dtype == BF16:
        assert w.dtype == np.uint16, "bf16 weights are passed as uint16 bit patterns"
        return w.astype(np.uint32)
    return np.ascontiguousarray(w, dtype=np.float32).view(np.uint32).copy()


def value_of(bits: np.ndarray, dtype: int) -> np.ndarray:
    """Bit patterns -> float64 values (exact)."""
    b = np.asarray(bits).astype(np.uint32)
    if dtype == BF16:
        b = b << np.uint32(16)
    return b.view(np.float32).astype(np.float64)


# ------------------------------------------------------------------ scalar API
def splitmix64(x: int) -> int:
    return lib().uo_splitmix64(x)


def hash_index(kind, seed, layer, t, row, p, ncols) -> int:
    return lib().uo_hash_index(kind, seed, layer, t, row, p, ncols)


def hash_indices(kind, seed, layer, t, M, positions, ncols) -> np.ndarray:
    """[M, n] index table for positions (loops in Python over the C scalar hash)."""
    L = lib()
    return np.array([[L.uo_hash_index(kind, seed, layer, t, i, int(p), ncols) for p in positions]
                     for i in range(M)], dtype=np.int64)


def update(dtype, cell_bits, x_bits) -> int:
    return lib().uo_update(dtype, cell_bits, x_bits)


def retrieve(dtype, bonded_bits) -> int:
    b = np.ascontiguousarray(bonded_bits, dtype=np.uint32)
    return lib().uo_retrieve(dtype, _ptr(b), len(b))


def sketch_unit(w_bits, positions, M, N, dtype=F32, hash_kind=HASH_X, seed=0, layer=0, t=0):
    w = np.ascontiguousarray(w_bits, dtype=np.uint32)
    p = np.ascontiguousarray(positions, dtype=np.uint32)
    cells = np.zeros(M * N, dtype=np.uint32)
    _check(lib().uo_sketch_unit(dtype, _ptr(w), _ptr(p), len(w), hash_kind, seed, layer, t, M, N,
                                _ptr(cells)), "sketch_unit")
    return cells.reshape(M, N)


def retrieve_unit(cells, positions, dtype=F32, hash_kind=HASH_X, seed=0, layer=0, t=0):
    cells = np.ascontiguousarray(cells, dtype=np.uint32)
    M, N = cells.shape
    p = np.ascontiguousarray(positions, dtype=np.uint32)
    out = np.zeros(len(p), dtype=np.uint32)
    _check(lib().uo_retrieve_unit(dtype, _ptr(cells), hash_kind, seed, layer, t, M, N, _ptr(p), len(p),
                                  _ptr(out)), "retrieve_unit")
    return out


def importance(A: np.ndarray) -> np.ndarray:
    """Eq. 7: I_j = (1/N) sum_k a_kj^2 (fp64)."""
    A = np.ascontiguousarray(A, dtype=np.float32)
    N, d = A.shape
    out = np.zeros(d, dtype=np.float64)
    _check(lib().uo_importance(_ptr(A), N, d, _ptr(out)), "importance")
    return out


def allocate(scores, T, C=None, M=1, min_cols=1, lengths=None):
    """Per-unit columns for unit scores under a budget of T cells (C defaults to U).  M: the sketch
    rows of every class, or a sequence of C per-class row counts (ledger L30)."""
    s = np.ascontiguousarray(scores, dtype=np.float64)
    U = len(s)
    C = U if C is None else C
    Mc = np.full(C, M, dtype=np.int32) if np.isscalar(M) else np.ascontiguousarray(M, dtype=np.int32)
    assert len(Mc) == C
    L_u = np.ones(U, dtype=np.uint64) if lengths is None else np.ascontiguousarray(lengths, dtype=np.uint64)
    cls = np.zeros(U, dtype=np.uint8)
    ncols = np.zeros(U, dtype=np.int32)
    _check(lib().uo_allocate(U, _ptr(s), _ptr(L_u), T, C, _ptr(Mc), min_cols, _ptr(cls), _ptr(ncols)), "allocate")
    return ncols, cls


# ------------------------------------------------------------------ model plan
@dataclass
class Plan:
    shapes: list            # [(out, in)]
    dtype: int
    M: int
    gran: int
    g: int
    C: int
    min_cols: int
    hash_kind: int
    seed: int
    unit_base: np.ndarray   # [L+1]
    cls: np.ndarray         # [U]
    ncols: np.ndarray       # [U]
    offsets: np.ndarray     # [U+1] cells
    acct: np.ndarray        # [L, 4] budget bits, class-map bits, T, achieved bits
    state_bits: int = 0     # 0: raw states in the weight dtype; 4 / 8: stacked quantisation
    group: int = 128        # cells per quantisation group (layers start at multiples of it)
    variant: int = 0        # ABSMAXMIN (the paper's sketch), ABSMINMAX, COUNTMIN (App. C.2)
    topk: int = 0           # Top-K outliers per layer stored apart (App. A)
    nrows: np.ndarray = None  # [U] sketch rows per unit (its class's; ledger L30)
    class_rows: tuple = None  # per-class rows, or None (every class has M)
    extra: dict = field(default_factory=dict)

    @property
    def total_cells(self) -> int:
        end = int(self.offsets[-1])
        return end if not self.state_bits else -(-end // self.group) * self.group

    def layer_units(self, l):
        return int(self.unit_base[l]), int(self.unit_base[l + 1])

    def layer_slices(self, l):
        u0, u1 = self.layer_units(l)
        return (np.ascontiguousarray(self.ncols[u0:u1]), np.ascontiguousarray(self.offsets[u0:u1 + 1]),
                np.ascontiguousarray(self.nrows[u0:u1]))


def plan(shapes, bpw, M=3, dtype=BF16, saliency=None, gran=GRAN_ROW, g=1, C=None, min_cols=1,
         hash_kind=HASH_X, seed=0, state_bits=0, group=128, variant=ABSMAXMIN, layer_importance=None,
         topk=0, class_rows=None) -> Plan:
    L = len(shapes)
    outf = np.array([s[0] for s in shapes], dtype=np.int64)
    inf = np.array([s[1] for s in shapes], dtype=np.int64)
    if C is None:
        C = 4 if saliency is not None and gran != GRAN_OUTROW else 1
    sal_arrays = None
    sal_ptrs = None
    if saliency is not None:
        sal_arrays = [None if s is None else np.ascontiguousarray(s, dtype=np.float32) for s in saliency]
        sal_ptrs = (ct.c_void_p * L)(*[None if a is None else a.ctypes.data for a in sal_arrays])
    U = int(np.sum(inf // g)) if gran == GRAN_ROW else int(np.sum(outf)) if gran == GRAN_OUTROW else L
    unit_base = np.zeros(L + 1, dtype=np.int64)
    cls = np.zeros(max(U, 1), dtype=np.uint8)
    ncols = np.zeros(max(U, 1), dtype=np.int32)
    offsets = np.zeros(max(U, 1) + 1, dtype=np.int64)
    acct = np.zeros(4 * L, dtype=np.int64)
    limp = None if layer_importance is None else np.ascontiguousarray(layer_importance, dtype=np.float64)
    crows = None
    if class_rows is not None:
        crows = np.ascontiguousarray(class_rows, dtype=np.int32)
        if len(crows) != C:
            raise OracleError(EINVAL, "plan: class_rows needs one row count per class")
    nrows = np.zeros(max(U, 1), dtype=np.uint8)
    # USK-XG plans score each ROW unit by its key group's mean importance (ledger L33)
    score_group = KEY_GROUP if (hash_kind == HASH_XG and gran == GRAN_ROW) else 1
    st = lib().uo_plan2(L, _ptr(outf), _ptr(inf), dtype,
                        ct.cast(sal_ptrs, ct.c_void_p) if sal_ptrs is not None else None,
                        float(bpw), M, gran, g, C, min_cols, state_bits, group,
                        None if limp is None else _ptr(limp), int(topk), None if crows is None else _ptr(crows),
                        score_group, _ptr(unit_base), _ptr(cls), _ptr(ncols), _ptr(nrows), _ptr(offsets), _ptr(acct))
    _check(st, "plan")
    return Plan(list(map(tuple, zip(outf.tolist(), inf.tolist()))), dtype, M, gran, g, C, min_cols, hash_kind,
                seed, unit_base, cls[:U], ncols[:U], offsets[:U + 1], acct.reshape(L, 4), state_bits, group, variant,
                int(topk), nrows[:U], None if crows is None else tuple(int(v) for v in crows))


def layer_cells(importance, numel, units, M, min_cols, T) -> np.ndarray:
    """First level of the two-level allocation (ledger L28): cells per layer."""
    imp = np.ascontiguousarray(importance, dtype=np.float64)
    n = np.ascontiguousarray(numel, dtype=np.int64)
    u = np.ascontiguousarray(units, dtype=np.int64)
    out = np.zeros(len(imp), dtype=np.int64)
    _check(lib().uo_layer_cells(len(imp), _ptr(imp), _ptr(n), _ptr(u), M, min_cols, T, _ptr(out)), "layer_cells")
    return out


def _np_dtype(dtype):
    return np.uint16 if dtype == BF16 else np.uint32


def build_layer(pl: Plan, l: int, W: np.ndarray, sketch: np.ndarray, t_begin=0, t_end=None, exclude=None):
    """Build units [t_begin, t_end) of layer l from W ([out,in] raw bits: uint16 bf16 / float32)
    into the model sketch (raw cells, uint16 or uint32).  exclude: optional [out, in] bool mask of
    weights kept out of the sketch (Top-K outliers)."""
    out, inn = pl.shapes[l]
    u0, u1 = pl.layer_units(l)
    t_end = (u1 - u0) if t_end is None else t_end
    W = np.ascontiguousarray(W)
    if pl.dtype == F32:
        W = W.astype(np.float32, copy=False)
    assert W.shape == (out, inn)
    ncols, offs, nrows = pl.layer_slices(l)
    assert sketch.dtype == _np_dtype(pl.dtype) and sketch.flags["C_CONTIGUOUS"]
    ex = None if exclude is None else np.ascontiguousarray(exclude, dtype=np.uint8)
    _check(lib().uo_build_units(pl.dtype, _ptr(W), out, inn, l, pl.gran, pl.g, t_begin, t_end, _ptr(ncols),
                                _ptr(offs), _ptr(nrows), pl.hash_kind, pl.seed, _ptr(sketch), pl.variant,
                                None if ex is None else _ptr(ex)), "build_units")


def topk(dtype, W: np.ndarray, K: int):
    """Top-K outliers of W (App. A): flat indices (ascending) and raw bits of the K weights of
    largest |w| (ties -> smaller flat index)."""
    Wb = np.ascontiguousarray(W, dtype=_np_dtype(dtype)) if dtype == BF16 else \
        np.ascontiguousarray(W, dtype=np.float32).view(np.uint32)
    n = Wb.size
    idx = np.zeros(max(K, 1), dtype=np.int64)
    vals = np.zeros(max(K, 1), dtype=np.uint32)
    _check(lib().uo_topk(dtype, _ptr(Wb), n, K, _ptr(idx), _ptr(vals)), "topk")
    return idx[:K], vals[:K]


@dataclass
class TSketch:
    """A sketch with Top-K outlier side tables: raw cells + per layer (flat indices, raw bits)."""
    cells: np.ndarray
    idx: list
    vals: list


@dataclass
class QSketch:
    """A quantised sketch (state_bits 4 / 8): int8 codes per cell, fp32 scales per group, the
    packed code bytes as stored, and the dequantised fp32 cells (bit patterns) used for
    retrieval."""
    codes: np.ndarray       # int8 [total_cells]
    scales: np.ndarray      # float32 [total_cells / group]
    packed: np.ndarray      # uint8 code storage
    deq: np.ndarray         # uint32 fp32 bits [total_cells]
    raw: np.ndarray         # the raw (pre-quantisation) states, weight dtype


def inf_bits(dtype):
    return 0x7F80 if dtype == BF16 else 0x7F800000


def quantize(dtype, raw: np.ndarray, q: int, G: int):
    """SPEC quant: per-group fp32 absmax scale, round-half-away codes; (codes int8, scales f32)."""
    raw = np.ascontiguousarray(raw, dtype=_np_dtype(dtype))
    n = len(raw)
    codes = np.zeros(n, dtype=np.int8)
    scales = np.zeros(n // G, dtype=np.float32)
    _check(lib().uo_quantize(dtype, _ptr(raw), n, q, G, _ptr(codes), _ptr(scales)), "quantize")
    return codes, scales


def dequantize(codes: np.ndarray, scales: np.ndarray, G: int) -> np.ndarray:
    """fp32 bits of fl32(code * scale) per cell."""
    codes = np.ascontiguousarray(codes, dtype=np.int8)
    scales = np.ascontiguousarray(scales, dtype=np.float32)
    out = np.zeros(len(codes), dtype=np.uint32)
    _check(lib().uo_dequantize(G, _ptr(codes), _ptr(scales), len(codes), _ptr(out)), "dequantize")
    return out


def pack_codes(q: int, codes: np.ndarray) -> np.ndarray:
    codes = np.ascontiguousarray(codes, dtype=np.int8)
    out = np.zeros(len(codes) * q // 8, dtype=np.uint8)
    _check(lib().uo_pack_codes(q, _ptr(codes), len(codes), _ptr(out)), "pack_codes")
    return out


def f32_to_bf16_rne(bits: np.ndarray) -> np.ndarray:
    L = lib()
    return np.array([L.uo_f32_to_bf16_rne(int(b)) for b in np.asarray(bits).ravel()],
                    dtype=np.uint16).reshape(np.shape(bits))


def build_model(pl: Plan, weights, layers=None):
    """Raw plans: the sketch cells (uint16 / uint32).  Quantised plans: a QSketch (raw states
    built into a +Inf-initialised buffer, then quantised per group)."""
    layers = range(len(weights)) if layers is None else layers
    if pl.topk:
        cells = np.zeros(pl.total_cells, dtype=_np_dtype(pl.dtype))
        idx, vals = [None] * len(pl.shapes), [None] * len(pl.shapes)
        for l, W in zip(layers, weights):
            out, inn = pl.shapes[l]
            idx[l], vals[l] = topk(pl.dtype, W, min(pl.topk, out * inn))
            mask = np.zeros(out * inn, dtype=bool)
            mask[idx[l]] = True
            build_layer(pl, l, W, cells, exclude=mask.reshape(out, inn))
        return TSketch(cells, idx, vals)
    if not pl.state_bits:
        sketch = np.zeros(pl.total_cells, dtype=_np_dtype(pl.dtype))
        for l, W in zip(layers, weights):
            build_layer(pl, l, W, sketch)
        return sketch
    raw = np.full(pl.total_cells, inf_bits(pl.dtype), dtype=_np_dtype(pl.dtype))
    for l, W in zip(layers, weights):
        build_layer(pl, l, W, raw)
    codes, scales = quantize(pl.dtype, raw, pl.state_bits, pl.group)
    return QSketch(codes, scales, pack_codes(pl.state_bits, codes), dequantize(codes, scales, pl.group), raw)


def _retrieval_view(pl: Plan, sketch):
    """(dtype, cells) on which Eq. 5 runs: raw cells, or the dequantised fp32 cells."""
    if isinstance(sketch, QSketch):
        return F32, sketch.deq
    if isinstance(sketch, TSketch):
        return pl.dtype, sketch.cells
    return pl.dtype, sketch


def _to_plan_dtype(pl: Plan, sketch, bits: np.ndarray) -> np.ndarray:
    if isinstance(sketch, QSketch) and pl.dtype == BF16:
        return f32_to_bf16_rne(bits)
    return bits


def reconstruct_rows(pl: Plan, sketch, l: int, o_begin=0, o_end=None) -> np.ndarray:
    """W' rows in the plan dtype (quantised plans: the dequantised value, RNE to bf16)."""
    out, inn = pl.shapes[l]
    o_end = out if o_end is None else o_end
    ncols, offs, nrows = pl.layer_slices(l)
    dt, cells = _retrieval_view(pl, sketch)
    res = np.zeros((o_end - o_begin, inn), dtype=_np_dtype(dt))
    _check(lib().uo_reconstruct_rows(dt, _ptr(cells), out, inn, l, pl.gran, pl.g, _ptr(ncols), _ptr(offs),
                                     _ptr(nrows), pl.hash_kind, pl.seed, o_begin, o_end, _ptr(res), pl.variant),
           "reconstruct_rows")
    if isinstance(sketch, TSketch):  # outliers keep their value (App. A)
        o_idx, j_idx = sketch.idx[l] // inn, sketch.idx[l] % inn
        sel = (o_idx >= o_begin) & (o_idx < o_end)
        res[o_idx[sel] - o_begin, j_idx[sel]] = sketch.vals[l][sel]
    return _to_plan_dtype(pl, sketch, res)


def reconstruct_entries(pl: Plan, sketch, l: int, oj: np.ndarray) -> np.ndarray:
    out, inn = pl.shapes[l]
    ncols, offs, nrows = pl.layer_slices(l)
    dt, cells = _retrieval_view(pl, sketch)
    oj = np.ascontiguousarray(oj, dtype=np.int64)
    res = np.zeros(len(oj), dtype=np.uint32)
    _check(lib().uo_reconstruct_entries(dt, _ptr(cells), out, inn, l, pl.gran, pl.g, _ptr(ncols),
                                        _ptr(offs), _ptr(nrows), pl.hash_kind, pl.seed, _ptr(oj), len(oj), _ptr(res),
                                        pl.variant), "reconstruct_entries")
    if isinstance(sketch, TSketch):
        flat = oj[:, 0] * inn + oj[:, 1]
        pos = np.searchsorted(sketch.idx[l], flat)
        hit = (pos < len(sketch.idx[l])) & (sketch.idx[l][np.minimum(pos, len(sketch.idx[l]) - 1)] == flat)
        res[hit] = sketch.vals[l][pos[hit]]
    return _to_plan_dtype(pl, sketch, res).astype(np.uint32)


def linear_rows(pl: Plan, sketch, l: int, x: np.ndarray, o_begin=0, o_end=None) -> np.ndarray:
    """fp64 y[T, o_end-o_begin] = x[T, in] @ W'[o_begin:o_end]^T (quantised plans: W' = the
    dequantised fp32 values, not rounded to the weight dtype)."""
    out, inn = pl.shapes[l]
    o_end = out if o_end is None else o_end
    x = np.ascontiguousarray(np.atleast_2d(x), dtype=np.float64)
    T = x.shape[0]
    if isinstance(sketch, TSketch):  # fp64 matmul of the overlaid W' (uo_linear_rows is pinned to it)
        return x @ value_of(reconstruct_rows(pl, sketch, l, o_begin, o_end), pl.dtype).T
    ncols, offs, nrows = pl.layer_slices(l)
    dt, cells = _retrieval_view(pl, sketch)
    y = np.zeros((T, o_end - o_begin), dtype=np.float64)
    _check(lib().uo_linear_rows(dt, _ptr(cells), out, inn, l, pl.gran, pl.g, _ptr(ncols), _ptr(offs), _ptr(nrows),
                                pl.hash_kind, pl.seed, _ptr(x), T, o_begin, o_end, _ptr(y), pl.variant), "linear_rows")
    return y


def aggregate_grad(pl: Plan, l: int, grad: np.ndarray) -> np.ndarray:
    """Aggregated-gradient baseline (Figure 4a): per cell of layer l, the 2^-48 fixed-point sum of
    the gradients of the weights mapped to it in each sketch row (ledger L26).  grad: [out, in]
    values (any float dtype, exact in fp64)."""
    out, inn = pl.shapes[l]
    ncols, offs, nrows = pl.layer_slices(l)
    g = np.ascontiguousarray(grad, dtype=np.float64)
    assert g.shape == (out, inn)
    res = np.zeros(int(offs[-1] - offs[0]), dtype=np.float32)
    _check(lib().uo_aggregate_grad(_ptr(g), out, inn, l, pl.gran, pl.g, len(ncols), _ptr(ncols), _ptr(offs), _ptr(nrows),
                                   pl.hash_kind, pl.seed, _ptr(res)), "aggregate_grad")
    return res


STATS_KEYS = ("weights", "untouched", "sign_errors", "zero_weights", "rel_exact", "rel_lt_1e-3", "rel_1e-3",
              "rel_1e-2", "rel_1e-1", "rel_1", "rel_ge_10", "cells", "unoccupied")


def stats(pl: Plan, l: int, W: np.ndarray, Wp: np.ndarray) -> dict:
    """Compression report of layer l (ledger L27): counts keyed by STATS_KEYS."""
    out, inn = pl.shapes[l]
    ncols, offs, nrows = pl.layer_slices(l)
    W = np.ascontiguousarray(W, dtype=_np_dtype(pl.dtype) if pl.dtype == BF16 else np.float32)
    Wp = np.ascontiguousarray(Wp)
    if pl.dtype == F32:
        W = W.view(np.uint32)
        Wp = Wp.view(np.uint32) if Wp.dtype != np.uint32 else Wp
    counts = np.zeros(13, dtype=np.int64)
    _check(lib().uo_stats(pl.dtype, _ptr(W), _ptr(Wp), out, inn, l, pl.gran, pl.g, len(ncols), _ptr(ncols), _ptr(offs),
                          _ptr(nrows), pl.hash_kind, pl.seed, _ptr(counts)), "stats")
    return dict(zip(STATS_KEYS, counts.tolist()))


def peak_memory(layer_bytes, sketch_bytes) -> int:
    a = np.ascontiguousarray(layer_bytes, dtype=np.int64)
    b = np.ascontiguousarray(sketch_bytes, dtype=np.int64)
    return lib().uo_peak_memory(_ptr(a), _ptr(b), len(a))
