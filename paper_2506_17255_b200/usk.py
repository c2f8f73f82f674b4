"""Thin Python binding of libusk (include/usk.h) -- argument marshalling only.

Every step of the sketch path runs in the CUDA kernels of ``libusk.so``; this module only turns
torch tensors into pointers/sizes and raises on non-zero status.  PyTorch is used for device
memory and streams.  There is NO CPU fallback: importing this module without the built
library raises.
"""
from __future__ import annotations

import ctypes as ct
import os
from dataclasses import dataclass

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libusk.so")

OK, EINVAL, ESHAPE, EBUDGET, ENONFINITE, ECUDA, EUNSUPPORTED, ERANGE = range(8)
F32, BF16 = 0, 1
GRAN = {"row": 0, "layer": 1, "outrow": 2}
HASH = {"x": 0, "identity": 1, "xg": 2}
LAYOUT = {"unit_major": 0, "query": 1}
VARIANT = {"absmaxmin": 0, "absminmax": 1, "countmin": 2}
STATS_KEYS = ("weights", "untouched", "sign_errors", "zero_weights", "rel_exact", "rel_lt_1e-3", "rel_1e-3",
              "rel_1e-2", "rel_1e-1", "rel_1", "rel_ge_10", "cells", "unoccupied")
DTYPE = {"f32": F32, "fp32": F32, "float32": F32, "bf16": BF16, "bfloat16": BF16}


class UskError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_STATUS.get(status, status)}: {msg}")
        self.status = status


_STATUS = {0: "USK_OK", 1: "USK_EINVAL", 2: "USK_ESHAPE", 3: "USK_EBUDGET", 4: "USK_ENONFINITE", 5: "USK_ECUDA",
           6: "USK_EUNSUPPORTED", 7: "USK_ERANGE"}


class _Shape(ct.Structure):
    _fields_ = [("out_features", ct.c_int64), ("in_features", ct.c_int64)]


class _Params(ct.Structure):
    _fields_ = [("bpw", ct.c_double), ("rows", ct.c_int32), ("granularity", ct.c_int32),
                ("dims_per_unit", ct.c_int32), ("n_classes", ct.c_int32), ("min_cols", ct.c_int32),
                ("hash", ct.c_int32), ("dtype", ct.c_int32), ("seed", ct.c_uint64), ("state_bits", ct.c_int32),
                ("group_size", ct.c_int32), ("variant", ct.c_int32), ("layer_importance", ct.c_void_p),
                ("topk", ct.c_int64), ("class_rows", ct.c_void_p), ("layout", ct.c_int32), ("reserved", ct.c_int32)]


class _PlanInfo(ct.Structure):
    _fields_ = [("n_layers", ct.c_int32), ("rows", ct.c_int32), ("n_classes", ct.c_int32), ("dtype", ct.c_int32),
                ("n_units", ct.c_int64), ("total_cells", ct.c_int64), ("sketch_bytes", ct.c_int64),
                ("numel", ct.c_int64), ("budget_bits", ct.c_int64), ("achieved_bits", ct.c_int64),
                ("state_bits", ct.c_int32), ("group_size", ct.c_int32), ("n_groups", ct.c_int64),
                ("scales_offset", ct.c_int64), ("topk", ct.c_int64), ("layout", ct.c_int32), ("hash", ct.c_int32)]


class _LayerInfo(ct.Structure):
    _fields_ = [("out_features", ct.c_int64), ("in_features", ct.c_int64), ("unit_begin", ct.c_int64),
                ("n_units", ct.c_int64), ("cell_begin", ct.c_int64), ("n_cells", ct.c_int64),
                ("budget_bits", ct.c_int64), ("meta_bits", ct.c_int64), ("cells_T", ct.c_int64),
                ("achieved_bits", ct.c_int64), ("n_outliers", ct.c_int64), ("outlier_offset", ct.c_int64),
                ("qbyte_begin", ct.c_int64), ("qbytes", ct.c_int64), ("qchunk_units", ct.c_int32),
                ("reserved", ct.c_int32)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2506_17255_b200.build` "
                          "(or __graft_entry__.build()); there is no fallback path")
    L = ct.CDLL(LIB_PATH)
    p, i32, i64, u64 = ct.c_void_p, ct.c_int32, ct.c_int64, ct.c_uint64
    sig = {
        "usk_importance": (i32, [p, i32, i64, i64, p, p]),
        "usk_plan_allocation": (i32, [ct.POINTER(_Shape), i32, p, ct.POINTER(_Params), ct.POINTER(p), p]),
        "usk_plan_query": (i32, [p, ct.POINTER(_PlanInfo)]),
        "usk_plan_layer": (i32, [p, i32, ct.POINTER(_LayerInfo)]),
        "usk_plan_export": (i32, [p, i32, p, p, p, p]),
        "usk_build": (i32, [p, p, p, i32, p, p]),
        "usk_build_rows": (i32, [p, i32, i64, i64, p, p, p]),
        "usk_reconstruct": (i32, [p, p, i32, i64, i64, p, i64, p]),
        "usk_prefetch_l2": (i32, [p, p, i32, i32, p]),
        "usk_reconstruct_batch": (i32, [p, p, p, i32, p, p, p]),
        "usk_linear_workspace_bytes": (ct.c_size_t, [p, i32, i64, i64, i64]),
        "usk_linear": (i32, [p, p, i32, p, i32, i64, p, i32, i64, i64, p, ct.c_size_t, p]),
        "usk_linear_batch_workspace_bytes": (ct.c_size_t, [p, p, p, i32]),
        "usk_linear_batch": (i32, [p, p, p, p, i32, p, i32, p, i32, p, ct.c_size_t, p]),
        "usk_linear_batch_tokens_workspace_bytes": (ct.c_size_t, [p, p, p, i32, i64]),
        "usk_linear_batch_tokens": (i32, [p, p, p, p, i32, p, i32, i64, p, i32, p, ct.c_size_t, p]),
        "usk_gemm_tokens": (i32, [p, i64, i64, p, p, i32, p, i32, p]),
        "usk_check": (i32, [p, p]),
        "usk_plan_destroy": (None, [p]),
        "usk_status_string": (ct.c_char_p, [i32]),
        "usk_last_error": (ct.c_char_p, []),
        "usk_launch_count": (i64, [i32]),
        "usk_aggregate_grad_workspace_bytes": (ct.c_size_t, [p, i32]),
        "usk_stats_workspace_bytes": (ct.c_size_t, [p, i32]),
        "usk_stats": (i32, [p, p, i32, p, p, p, ct.c_size_t, p]),
        "usk_aggregate_grad": (i32, [p, i32, p, i32, p, p, ct.c_size_t, p]),
        "usk_trace_read": (i32, [p, i64, p, i32]),
        "usk_linear_batch_peers": (i32, [p, p, p, p, i32, p, i32, i32, p, p, ct.c_size_t, p]),
        "usk_peer_wait": (i32, [p, p, p]),
        "usk_trace_reset": (None, []),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    return L


lib = _load()


def _check(st: int):
    if st != OK:
        raise UskError(st, lib.usk_last_error().decode())


def _stream(stream):
    import torch
    if stream is None:
        if not torch.cuda.is_available():
            return ct.c_void_p(0)  # host-side validation still runs; device work reports USK_ECUDA
        stream = torch.cuda.current_stream()
    return ct.c_void_p(stream.cuda_stream)


def _ptr(t):
    return ct.c_void_p(t.data_ptr()) if t is not None else ct.c_void_p(0)


def _need(t, what: str, shape=None, dtype=None, contiguous: bool = True):
    """Argument marshalling guard: the C ABI takes raw pointers with an implied dense row-major
    layout, so a strided view or a wrong dtype would be silently reinterpreted."""
    import torch
    if contiguous and not t.is_contiguous():
        raise UskError(EINVAL, f"{what}: tensor must be contiguous (got strides {tuple(t.stride())})")
    if dtype is not None:
        want = torch.bfloat16 if dtype == BF16 else torch.float32
        if t.dtype != want:
            raise UskError(EINVAL, f"{what}: dtype {t.dtype}, the plan needs {want}")
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise UskError(ESHAPE, f"{what}: shape {tuple(t.shape)}, expected {tuple(shape)}")


def _dtype_code(t) -> int:
    import torch
    if t.dtype == torch.bfloat16:
        return BF16
    if t.dtype == torch.float32:
        return F32
    raise UskError(EINVAL, f"unsupported tensor dtype {t.dtype}")


@dataclass
class LayerInfo:
    out_features: int
    in_features: int
    unit_begin: int
    n_units: int
    cell_begin: int
    n_cells: int
    budget_bits: int
    meta_bits: int
    cells_T: int
    achieved_bits: int
    n_outliers: int = 0
    outlier_offset: int = 0
    qbyte_begin: int = 0
    qbytes: int = 0
    qchunk_units: int = 0
    reserved: int = 0


class Plan:
    """Owns a usk_plan handle (destroyed on garbage collection)."""

    def __init__(self, handle: ct.c_void_p, shapes, dtype: int):
        self.handle = handle
        self.shapes = [tuple(s) for s in shapes]
        self.dtype = dtype
        info = _PlanInfo()
        _check(lib.usk_plan_query(handle, ct.byref(info)))
        self.info = {k: getattr(info, k) for k, _ in _PlanInfo._fields_}
        self.layers = []
        for l in range(len(shapes)):
            li = _LayerInfo()
            _check(lib.usk_plan_layer(handle, l, ct.byref(li)))
            self.layers.append(LayerInfo(*[getattr(li, k) for k, _ in _LayerInfo._fields_]))

    @property
    def sketch_bytes(self) -> int:
        return self.info["sketch_bytes"]

    def new_sketch(self, device=None):
        import torch
        return torch.empty(self.sketch_bytes, dtype=torch.uint8, device=device or "cuda")

    def export(self, layer: int):
        import numpy as np
        n = self.layers[layer].n_units
        cls = np.zeros(n, np.uint8)
        ncols = np.zeros(n, np.int32)
        nrows = np.zeros(n, np.uint8)
        offs = np.zeros(n + 1, np.int64)
        _check(lib.usk_plan_export(self.handle, layer, cls.ctypes.data, ncols.ctypes.data, nrows.ctypes.data,
                                   offs.ctypes.data))
        return cls, ncols, nrows, offs

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value and lib is not None:
            lib.usk_plan_destroy(h)
            self.handle = None


def plan_allocation(shapes, *, bpw: float, rows: int = 3, granularity: str = "row", dims_per_unit: int = 1,
                    n_classes: int = 0, min_cols: int = 1, hash: str = "x", dtype: str = "bf16", seed: int = 0,
                    saliency=None, state_bits: int = 0, group_size: int = 0, variant: str = "absmaxmin",
                    layer_importance=None, topk: int = 0, class_rows=None, layout: str = "unit_major",
                    stream=None) -> Plan:
    """usk_plan_allocation. saliency: None or list of (None | float32 CUDA tensor [in_features]).
    state_bits 4 / 8: stacked state quantisation with group_size cells per scale (0 = 128).
    class_rows: None or the sketch rows of each importance class (ledger L30).
    hash "xg" + layout "query": the packed decode layout (usk.h USK_LAYOUT_QUERY, ledger L32)."""
    n = len(shapes)
    arr = (_Shape * n)(*[_Shape(int(o), int(i)) for (o, i) in shapes])
    prm = _Params(float(bpw), rows, GRAN[granularity], dims_per_unit, n_classes, min_cols, HASH[hash],
                  DTYPE[dtype], seed & (2**64 - 1), state_bits, group_size, VARIANT[variant], None, int(topk), None,
                  LAYOUT[layout], 0)
    limp = None
    if layer_importance is not None:  # host doubles, kept alive for the call
        limp = (ct.c_double * n)(*[float(v) for v in layer_importance])
        prm.layer_importance = ct.cast(limp, ct.c_void_p)
    crows = None
    if class_rows is not None:  # host int32 [n_classes], kept alive for the call
        n_cls = n_classes if n_classes > 0 else (4 if saliency is not None and granularity != "outrow" else 1)
        if len(class_rows) != n_cls:
            raise UskError(1, f"class_rows needs one row count per class ({n_cls})")
        crows = (ct.c_int32 * len(class_rows))(*[int(v) for v in class_rows])
        prm.class_rows = ct.cast(crows, ct.c_void_p)
    sal = ct.c_void_p(0)
    keep = None
    if saliency is not None:
        keep = (ct.c_void_p * n)(*[None if s is None else s.data_ptr() for s in saliency])
        sal = ct.cast(keep, ct.c_void_p)
    h = ct.c_void_p(0)
    _check(lib.usk_plan_allocation(arr, n, sal, ct.byref(prm), ct.byref(h), _stream(stream)))
    return Plan(h, shapes, DTYPE[dtype])


def build(plan: Plan, weights, sketch, layer_ids=None, stream=None):
    import torch
    n = len(weights)
    want = torch.bfloat16 if plan.dtype == BF16 else torch.float32
    shapes = plan.shapes
    ptrs = [0] * n
    for k, w in enumerate(weights):  # one cheap pass; the detailed message only on a mismatch
        l = k if layer_ids is None else layer_ids[k]
        if 0 <= l < len(shapes) and (w.dtype != want or w.shape != shapes[l] or not w.is_contiguous()):
            _need(w, f"build: weights[{k}]", shapes[l], plan.dtype)
        ptrs[k] = w.data_ptr()
    wp = (ct.c_void_p * n)(*ptrs)
    ids = None if layer_ids is None else (ct.c_int32 * n)(*layer_ids)
    _check(lib.usk_build(plan.handle, wp, ids, n, _ptr(sketch), _stream(stream)))


def build_rows(plan: Plan, layer: int, row_begin: int, row_end: int, w_rows, sketch, stream=None):
    """usk_build_rows (output-row units): build only the units of rows [row_begin, row_end) of `layer`
    from w_rows = those rows of its [out, in] weight (a rank's shard)."""
    if 0 <= layer < len(plan.shapes):
        _need(w_rows, "build_rows: w_rows", (row_end - row_begin, plan.shapes[layer][1]), plan.dtype)
    _check(lib.usk_build_rows(plan.handle, layer, row_begin, row_end, _ptr(w_rows), _ptr(sketch), _stream(stream)))


def reconstruct(plan: Plan, sketch, layer: int, w_out, row_begin: int = 0, row_end=None, stream=None):
    row_end = plan.layers[layer].out_features if row_end is None else row_end
    _need(w_out, "reconstruct: w_out", dtype=plan.dtype, contiguous=False)
    if w_out.dim() != 2 or w_out.stride(1) != 1 or w_out.shape[0] < row_end - row_begin \
            or w_out.shape[1] < plan.shapes[layer][1]:
        raise UskError(ESHAPE, f"reconstruct: w_out must be [>= {row_end - row_begin}, {plan.shapes[layer][1]}] with "
                               f"unit column stride (got {tuple(w_out.shape)}, strides {tuple(w_out.stride())})")
    _check(lib.usk_reconstruct(plan.handle, _ptr(sketch), layer, row_begin, row_end, _ptr(w_out), w_out.stride(0),
                               _stream(stream)))


def reconstruct_batch(plan: Plan, sketch, layers, w_outs, stream=None):
    """usk_reconstruct_batch: whole layers (w_outs[k] = [out, >= in] row-major, unit column stride)."""
    n = len(layers)
    for k, (l, w) in enumerate(zip(layers, w_outs)):
        _need(w, f"reconstruct_batch: w_outs[{k}]", dtype=plan.dtype, contiguous=False)
        if 0 <= l < len(plan.shapes) and (w.dim() != 2 or w.stride(1) != 1 or w.shape[0] < plan.shapes[l][0]
                                          or w.shape[1] < plan.shapes[l][1]):
            raise UskError(ESHAPE, f"reconstruct_batch: w_outs[{k}] shape {tuple(w.shape)}")
    ids = (ct.c_int32 * n)(*layers)
    ptrs = (ct.c_void_p * n)(*[w.data_ptr() for w in w_outs])
    lds = (ct.c_int64 * n)(*[w.stride(0) for w in w_outs])
    _check(lib.usk_reconstruct_batch(plan.handle, _ptr(sketch), ids, n, ptrs, lds, _stream(stream)))


def prefetch_l2(plan: Plan, sketch, layer_begin: int = 0, layer_end=None, stream=None):
    """Warm the sketch bytes of layers [layer_begin, layer_end) into L2 (usk_prefetch_l2)."""
    layer_end = len(plan.layers) if layer_end is None else layer_end
    _check(lib.usk_prefetch_l2(plan.handle, _ptr(sketch), layer_begin, layer_end, _stream(stream)))


def linear_workspace_bytes(plan: Plan, layer: int, T: int = 1, out_begin: int = 0, out_end=None) -> int:
    out_end = plan.layers[layer].out_features if out_end is None else out_end
    return int(lib.usk_linear_workspace_bytes(plan.handle, layer, T, out_begin, out_end))


def new_workspace(plan: Plan, layer: int, T: int = 1, out_begin: int = 0, out_end=None, device=None):
    import torch
    return torch.zeros(max(linear_workspace_bytes(plan, layer, T, out_begin, out_end), 256), dtype=torch.uint8,
                       device=device or "cuda")


def linear(plan: Plan, sketch, layer: int, x, y, workspace, out_begin: int = 0, out_end=None, stream=None):
    """y[T, out_end-out_begin] = x[T, in] @ W'[out_begin:out_end]^T (x, y contiguous CUDA tensors)."""
    out_end = plan.layers[layer].out_features if out_end is None else out_end
    T = x.shape[0] if x.dim() == 2 else 1
    if 0 <= layer < len(plan.shapes):
        _need(x, "linear: x", (T, plan.shapes[layer][1]) if x.dim() == 2 else (plan.shapes[layer][1],))
        _need(y, "linear: y", (T, out_end - out_begin) if y.dim() == 2 else (out_end - out_begin,))
    _need(workspace, "linear: workspace")
    _check(lib.usk_linear(plan.handle, _ptr(sketch), layer, _ptr(x), _dtype_code(x), T, _ptr(y), _dtype_code(y),
                          out_begin, out_end, _ptr(workspace), workspace.numel() * workspace.element_size(),
                          _stream(stream)))


def _batch_args(layers, ranges):
    n = len(layers)
    ids = (ct.c_int32 * n)(*layers)
    rg = None if ranges is None else (ct.c_int64 * (2 * n))(*[v for r in ranges for v in r])
    return n, ids, rg


def linear_batch_workspace_bytes(plan: Plan, layers, ranges=None) -> int:
    n, ids, rg = _batch_args(layers, ranges)
    return int(lib.usk_linear_batch_workspace_bytes(plan.handle, ids, rg, n))


def new_batch_workspace(plan: Plan, layers, ranges=None, device=None):
    import torch
    return torch.zeros(max(linear_batch_workspace_bytes(plan, layers, ranges), 256), dtype=torch.uint8,
                       device=device or "cuda")


def linear_batch(plan: Plan, sketch, layers, x, ys, workspace, ranges=None, stream=None):
    """One launch for several T=1 sketch-GEMVs sharing x: ys[k] = x @ W'_{layers[k]}[range_k]^T."""
    n, ids, rg = _batch_args(layers, ranges)
    if len(ys) != n:
        raise UskError(ESHAPE, f"linear_batch: {len(ys)} outputs for {n} layers")
    _need(x, "linear_batch: x")
    for k, (l, y) in enumerate(zip(layers, ys)):
        if 0 <= l < len(plan.shapes):
            r = (0, plan.shapes[l][0]) if ranges is None else ranges[k]
            _need(y, f"linear_batch: ys[{k}]")
            if y.numel() != r[1] - r[0]:
                raise UskError(ESHAPE, f"linear_batch: ys[{k}] has {y.numel()} elements, range needs {r[1] - r[0]}")
    _need(workspace, "linear_batch: workspace")
    yp = (ct.c_void_p * n)(*[y.data_ptr() for y in ys])
    _check(lib.usk_linear_batch(plan.handle, _ptr(sketch), ids, rg, n, _ptr(x), _dtype_code(x), yp,
                                _dtype_code(ys[0]), _ptr(workspace), workspace.numel() * workspace.element_size(),
                                _stream(stream)))


def linear_batch_tokens_workspace_bytes(plan: Plan, layers, T: int, ranges=None) -> int:
    n, ids, rg = _batch_args(layers, ranges)
    return int(lib.usk_linear_batch_tokens_workspace_bytes(plan.handle, ids, rg, n, int(T)))


def linear_batch_tokens(plan: Plan, sketch, layers, x, ys, workspace, ranges=None, stream=None):
    """usk_linear_batch_tokens: T tokens (x [T, in] bf16) through several layers sharing x; the group's
    W' rows rebuilt once into the workspace, one tcgen05 GEMM; ys[k]: contiguous [T, rows_k]."""
    n, ids, rg = _batch_args(layers, ranges)
    if len(ys) != n:
        raise UskError(ESHAPE, f"linear_batch_tokens: {len(ys)} outputs for {n} layers")
    _need(x, "linear_batch_tokens: x")
    T = x.shape[0] if x.dim() == 2 else 1
    for k, (l, y) in enumerate(zip(layers, ys)):
        if 0 <= l < len(plan.shapes):
            r = (0, plan.shapes[l][0]) if ranges is None else ranges[k]
            _need(y, f"linear_batch_tokens: ys[{k}]")
            if y.numel() != T * (r[1] - r[0]):
                raise UskError(ESHAPE, f"linear_batch_tokens: ys[{k}] has {y.numel()} elements, needs {T * (r[1] - r[0])}")
    _need(workspace, "linear_batch_tokens: workspace")
    yp = (ct.c_void_p * n)(*[y.data_ptr() for y in ys])
    _check(lib.usk_linear_batch_tokens(plan.handle, _ptr(sketch), ids, rg, n, _ptr(x), _dtype_code(x), T, yp,
                                       _dtype_code(ys[0]), _ptr(workspace),
                                       workspace.numel() * workspace.element_size(), _stream(stream)))


def gemm_tokens(x, w, rows, ys, stream=None):
    """usk_gemm_tokens: the computation stage alone -- ys[k] = x @ w[block k]^T with the blocks of
    `rows` stacked in w (bf16 [sum rows, in], e.g. filled by reconstruct_batch); one GEMM."""
    _need(x, "gemm_tokens: x")
    _need(w, "gemm_tokens: w")
    n = len(rows)
    T = x.shape[0] if x.dim() == 2 else 1
    if len(ys) != n:
        raise UskError(ESHAPE, f"gemm_tokens: {len(ys)} outputs for {n} blocks")
    for k, y in enumerate(ys):
        _need(y, f"gemm_tokens: ys[{k}]")
        if y.numel() != T * rows[k]:
            raise UskError(ESHAPE, f"gemm_tokens: ys[{k}] has {y.numel()} elements, needs {T * rows[k]}")
    rw = (ct.c_int64 * n)(*rows)
    yp = (ct.c_void_p * n)(*[y.data_ptr() for y in ys])
    _check(lib.usk_gemm_tokens(_ptr(x), T, x.shape[-1], _ptr(w), rw, n, yp, _dtype_code(ys[0]), _stream(stream)))


class _Peers(ct.Structure):
    _fields_ = [("n_peers", ct.c_int32), ("my_rank", ct.c_int32), ("y_peer", ct.c_void_p), ("sig_peer", ct.c_void_p),
                ("epoch", ct.c_void_p)]


class Peers:
    """usk_peers (include/usk.h): the peer-mapped full-y pointers of every rank per layer of a grouped
    call, every rank's signal array, and this rank's device epoch counter.  Pointers are ints
    (device addresses valid in this process, e.g. torch symmetric-memory buffer_ptrs)."""

    def __init__(self, n_peers: int, my_rank: int, y_ptrs, sig_ptrs, epoch):
        n = len(y_ptrs[0])
        self._y = (ct.c_void_p * (n_peers * n))(*[int(y_ptrs[q][k]) for q in range(n_peers) for k in range(n)])
        self._s = (ct.c_void_p * n_peers)(*[int(v) for v in sig_ptrs])
        self.epoch = epoch
        self.c = _Peers(n_peers, my_rank, ct.cast(self._y, ct.c_void_p), ct.cast(self._s, ct.c_void_p),
                        ct.c_void_p(epoch.data_ptr()))


def linear_batch_peers(plan: Plan, sketch, layers, x, peers: Peers, workspace, ranges=None, y_dtype="f32", stream=None):
    """usk_linear_batch_peers: this rank's output ranges, stored into every rank's full y + flags."""
    n, ids, rg = _batch_args(layers, ranges)
    _need(x, "linear_batch_peers: x")
    _need(workspace, "linear_batch_peers: workspace")
    _check(lib.usk_linear_batch_peers(plan.handle, _ptr(sketch), ids, rg, n, _ptr(x), _dtype_code(x), DTYPE[y_dtype],
                                      ct.byref(peers.c), _ptr(workspace), workspace.numel() * workspace.element_size(),
                                      _stream(stream)))


def peer_wait(plan: Plan, peers: Peers, stream=None):
    """usk_peer_wait: wait until every rank's flag reached epoch + 1, then advance the epoch."""
    _check(lib.usk_peer_wait(plan.handle, ct.byref(peers.c), _stream(stream)))


def importance(A, out, stream=None):
    """Eq. 7: out[j] = mean_k A[k, j]^2 (A [N, d] bf16/fp32 CUDA, out float32 [d])."""
    _need(A, "importance: A")
    _need(out, "importance: out", (A.shape[1],), F32)
    _check(lib.usk_importance(_ptr(A), _dtype_code(A), A.shape[0], A.shape[1], _ptr(out), _stream(stream)))


def aggregate_grad(plan: Plan, layer: int, grad, cell_grad, workspace=None, stream=None):
    """usk_aggregate_grad: cell_grad[c] = fixed-point sum of grad over the weights mapped to cell c
    (aggregated-gradient baseline, Figure 4a).  cell_grad: float32 CUDA tensor [n_cells of layer]."""
    import torch
    if 0 <= layer < len(plan.shapes):
        _need(grad, "aggregate_grad: grad", plan.shapes[layer])
        _need(cell_grad, "aggregate_grad: cell_grad", (plan.layers[layer].n_cells,), F32)
    if workspace is None:
        workspace = torch.zeros(int(lib.usk_aggregate_grad_workspace_bytes(plan.handle, layer)), dtype=torch.uint8,
                                device=grad.device)
    _check(lib.usk_aggregate_grad(plan.handle, layer, _ptr(grad), _dtype_code(grad), _ptr(cell_grad), _ptr(workspace),
                                  workspace.numel(), _stream(stream)))
    return cell_grad


def stats(plan: Plan, sketch, layer: int, W, stream=None) -> dict:
    """usk_stats: the compression report of `layer` (counts keyed by STATS_KEYS)."""
    import torch
    if 0 <= layer < len(plan.shapes):
        _need(W, "stats: W", plan.shapes[layer], plan.dtype)
    counts = torch.zeros(13, dtype=torch.int64, device=W.device)
    ws = torch.zeros(int(lib.usk_stats_workspace_bytes(plan.handle, layer)), dtype=torch.uint8, device=W.device)
    _check(lib.usk_stats(plan.handle, _ptr(sketch), layer, _ptr(W), _ptr(counts), _ptr(ws), ws.numel(), _stream(stream)))
    return dict(zip(STATS_KEYS, counts.cpu().tolist()))


def check(plan: Plan, stream=None):
    _check(lib.usk_check(plan.handle, _stream(stream)))


def launch_count(reset: bool = False) -> int:
    return int(lib.usk_launch_count(1 if reset else 0))


def trace_read(max_launches: int = 4096, max_ctas: int = 1 << 18):
    """Tuning only (USK_TRACE=1): per launch, an int64 array [grid, 8] of %globaltimer stamps of
    every CTA (start, staged, compute done, exit; query kernels also: first bulk copy issued, first
    piece landed, first segment converted, griddepcontrol.wait returned), launches in issue order."""
    import numpy as np
    stamps = np.zeros(8 * max_ctas, np.uint64)
    grids = np.zeros(max_launches, np.int32)
    n = int(lib.usk_trace_read(stamps.ctypes.data, stamps.size, grids.ctypes.data, max_launches))
    out, c = [], 0
    for g in grids[:n]:
        out.append(stamps[8 * c:8 * (c + int(g))].astype(np.int64).reshape(int(g), 8))
        c += int(g)
    return out


def trace_reset():
    lib.usk_trace_reset()
