"""GPU parity of output-row units (SURVEY §8(f4) "Output-row units"; ledger L31): unit
(l, o) holds W[o, :] at positions p = j.  Plan arrays, sketch bytes and reconstructions bit-exact vs
the oracle; sketch-GEMV (one kernel per call, no cross-CTA reduction) within the 1e-5 bar, grouped
calls and output shards included; prefill within the bf16 bar; q4 states; the error cases."""
import numpy as np
import pytest

import synth
from test_gpu_parity import DT, assert_plan_equal, gemv_err, make_weights, sketch_cells, to_dev, w_bits

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def usk():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2506_17255_b200 import usk as u
    return u


CASES = [
    # (shapes, dtype, bpw, M, hash)
    ([(200, 2048), (72, 512)], "bf16", 0.5, 3, "x"),     # 1B-like rows (N = 21 at 2048 in), ragged row count
    ([(130, 8192)], "bf16", 0.5, 3, "x"),                 # down-projection rows (N = 85)
    ([(96, 264), (33, 136)], "bf16", 2.0, 3, "x"),         # ragged in (not a multiple of 32 / 128)
    ([(160, 512)], "f32", 2.0, 2, "x"),
    ([(64, 1024)], "bf16", 1.0, 1, "x"),
    ([(80, 640)], "bf16", 2.0, 5, "x"),                   # runtime-M
    ([(70, 256)], "bf16", 4.0, 3, "identity"),            # SPEC test hash
]
IDS = [f"{c[1]}-M{c[3]}-{c[4]}-{c[0][0][0]}x{c[0][0][1]}" for c in CASES]


def _x(i, seed, dtype):
    x = synth.vector(i, seed=seed)[0]
    if dtype == "bf16":
        xb = synth.f32_to_bf16_bits(x)
        return torch.from_numpy(xb.view(np.int16).copy()).view(torch.bfloat16).cuda(), \
            synth.bf16_bits_to_f32(xb).astype(np.float64)
    return torch.from_numpy(x).cuda(), x.astype(np.float64)


def _both(orc, usk, shapes, dtype, bpw, M, hk, **kw):
    Ws = make_weights(shapes, dtype, 31)
    pl = usk.plan_allocation(shapes, bpw=bpw, rows=M, granularity="outrow", dtype=dtype, seed=99, hash=hk, **kw)
    okw = dict(kw)
    if "group_size" in okw:
        okw["group"] = okw.pop("group_size")
    if "saliency" in okw and okw["saliency"] is not None:
        okw["saliency"] = [s.cpu().numpy() for s in okw["saliency"]]
    opl = orc.plan(shapes, bpw, M=M, dtype=DT[dtype], gran=orc.GRAN_OUTROW, seed=99,
                   hash_kind=0 if hk == "x" else 1, **okw)
    sk = pl.new_sketch()
    sk.fill_(0x77)
    dW = [to_dev(W, dtype) for W in Ws]
    usk.build(pl, dW, sk)
    usk.check(pl)
    return pl, opl, sk, orc.build_model(opl, Ws), Ws, dW


@pytest.mark.parametrize("case", CASES, ids=IDS)
def test_outrow_parity(orc, usk, case):
    shapes, dtype, bpw, M, hk = case
    pl, opl, sk, osk, Ws, dW = _both(orc, usk, shapes, dtype, bpw, M, hk)
    assert_plan_equal(pl, opl)
    np.testing.assert_array_equal(sketch_cells(sk, pl, dtype), osk)
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    for l, (o, i) in enumerate(shapes):
        Wr = torch.empty((o, i), dtype=tdt, device="cuda")
        usk.reconstruct(pl, sk, l, Wr)
        want = orc.reconstruct_rows(opl, osk, l)
        np.testing.assert_array_equal(w_bits(Wr, dtype), want)
        wv = orc.value_of(want, DT[dtype]).reshape(o, i)
        for xdt in (("bf16", "f32") if dtype == "bf16" else ("f32",)):
            xd, x64 = _x(i, 60 + l, xdt)
            y = torch.empty(o, dtype=torch.float32, device="cuda")
            usk.linear(pl, sk, l, xd.view(1, -1), y.view(1, -1), usk.new_workspace(pl, l))
            y64 = orc.linear_rows(opl, osk, l, x64)[0]
            assert gemv_err(y.cpu().numpy().astype(np.float64), y64, x64, wv) <= 1e-5
            y2 = torch.empty_like(y)
            usk.linear(pl, sk, l, xd.view(1, -1), y2.view(1, -1), usk.new_workspace(pl, l))
            assert torch.equal(y, y2)                                  # deterministic
            # an output shard: each row is computed by one warp from its own unit -> bitwise equal
            h = o // 3
            ys = torch.empty(o - h, dtype=torch.float32, device="cuda")
            usk.linear(pl, sk, l, xd.view(1, -1), ys.view(1, -1), usk.new_workspace(pl, l, 1, h, o), out_begin=h,
                       out_end=o)
            assert torch.equal(ys, y[h:])


def test_outrow_grouped_calls(orc, usk):
    """q|k|v (shared x) in one call: equal bits to the per-layer calls."""
    shapes = [(2048, 2048), (512, 2048), (512, 2048)]
    pl, opl, sk, osk, Ws, dW = _both(orc, usk, shapes, "bf16", 0.5, 3, "x")
    np.testing.assert_array_equal(sketch_cells(sk, pl, "bf16"), osk)
    x = synth.torch_vector(2048, 4, "cuda", torch.bfloat16)
    ys = [torch.empty(o, dtype=torch.float32, device="cuda") for o, _ in shapes]
    usk.linear_batch(pl, sk, [0, 1, 2], x.view(1, -1), [y.view(1, -1) for y in ys],
                     usk.new_batch_workspace(pl, [0, 1, 2]))
    x64 = x.float().cpu().numpy().astype(np.float64).ravel()
    rng = np.random.default_rng(1)
    for l, (o, i) in enumerate(shapes):
        y1 = torch.empty(o, dtype=torch.float32, device="cuda")
        usk.linear(pl, sk, l, x.view(1, -1), y1.view(1, -1), usk.new_workspace(pl, l))
        assert torch.equal(y1, ys[l])
        rs = rng.choice(o, 16, replace=False)
        for r in rs:
            y64 = orc.linear_rows(opl, osk, l, x64, int(r), int(r) + 1)[0]
            wv = orc.value_of(orc.reconstruct_rows(opl, osk, l, int(r), int(r) + 1), 1)
            assert gemv_err(ys[l][r:r + 1].cpu().numpy().astype(np.float64), y64, x64, wv) <= 1e-5


def test_outrow_prefill_and_q4(orc, usk):
    shapes = [(256, 512)]
    pl, opl, sk, osk, Ws, dW = _both(orc, usk, shapes, "bf16", 1.0, 3, "x")
    T = 96
    X = synth.torch_vector(512, 8, "cuda", torch.bfloat16, T=T)
    Y = torch.empty((T, 256), dtype=torch.bfloat16, device="cuda")
    usk.linear(pl, sk, 0, X, Y, usk.new_workspace(pl, 0, T))
    x64 = X.float().cpu().numpy().astype(np.float64)
    wv = orc.value_of(orc.reconstruct_rows(opl, osk, 0), 1).reshape(256, 512)
    scale = np.maximum(np.abs(x64) @ np.abs(wv).T, 1e-30)
    assert float(np.max(np.abs(Y.float().cpu().numpy() - orc.linear_rows(opl, osk, 0, x64)) / scale)) <= 2e-2
    # q4 states on output-row units
    pq, oq, skq, oskq, Wq, dWq = _both(orc, usk, [(96, 1024)], "bf16", 0.5, 3, "x", state_bits=4, group_size=128)
    Wr = torch.empty((96, 1024), dtype=torch.bfloat16, device="cuda")
    usk.reconstruct(pq, skq, 0, Wr)
    np.testing.assert_array_equal(w_bits(Wr, "bf16"), orc.reconstruct_rows(oq, oskq, 0))


def test_outrow_layer_importance(orc, usk):
    shapes = [(128, 512), (64, 1024), (96, 256)]
    pl, opl, sk, osk, Ws, dW = _both(orc, usk, shapes, "bf16", 1.0, 3, "x", layer_importance=[4.0, 1.0, 2.0])
    assert_plan_equal(pl, opl)
    np.testing.assert_array_equal(sketch_cells(sk, pl, "bf16"), osk)


def test_outrow_errors(usk):
    with pytest.raises(usk.UskError):
        usk.plan_allocation([(64, 64)], bpw=2.0, granularity="outrow", n_classes=2)
    with pytest.raises(usk.UskError):
        usk.plan_allocation([(64, 64)], bpw=2.0, granularity="outrow", dims_per_unit=2)
    with pytest.raises(usk.UskError):
        usk.plan_allocation([(64, 64)], bpw=2.0, granularity="outrow", topk=4)


@pytest.mark.parametrize("world", [2, 3])
def test_outrow_row_sharded_build_and_decode(orc, usk, world):
    """usk_build_rows: each 'rank' (run one after another on this GPU -- no rank waits on another)
    builds only its output shard from only its rows; the union of the shards is byte-identical to
    the full build and the oracle, and each rank's decode of its range from a sketch holding ONLY
    its own units equals the full call's rows bit for bit (no replication step)."""
    from paper_2506_17255_b200 import dist as udist
    shapes = [(200, 2048), (130, 8192), (96, 264)]
    pl, opl, sk, osk, Ws, dW = _both(orc, usk, shapes, "bf16", 0.5, 3, "x")
    full = sketch_cells(sk, pl, "bf16").copy()
    np.testing.assert_array_equal(full, osk)
    union = pl.new_sketch()
    union.fill_(0x33)
    for r in range(world):
        own = pl.new_sketch()
        own.fill_(0x44)                                            # this rank's sketch: only its units
        for l, (o, i) in enumerate(shapes):
            o0, o1 = udist.output_shard(o, r, world)
            rows_only = dW[l][o0:o1].contiguous()                 # the rank holds only its rows
            udist.build_output_shard(usk, pl, l, rows_only, own, r, world, rows_only=True)
            udist.build_output_shard(usk, pl, l, dW[l], union, r, world)
            x = synth.torch_vector(i, 30 + l, "cuda", torch.bfloat16)
            y_full = torch.empty(o, dtype=torch.float32, device="cuda")
            usk.linear(pl, sk, l, x.view(1, -1), y_full.view(1, -1), usk.new_workspace(pl, l))
            y_sh = torch.empty(o1 - o0, dtype=torch.float32, device="cuda")
            usk.linear(pl, own, l, x.view(1, -1), y_sh.view(1, -1), usk.new_workspace(pl, l, 1, o0, o1),
                       out_begin=o0, out_end=o1)
            assert torch.equal(y_sh, y_full[o0:o1])
        usk.check(pl)
    np.testing.assert_array_equal(sketch_cells(union, pl, "bf16"), full)


def test_build_rows_errors(usk):
    pl = usk.plan_allocation([(64, 64)], bpw=2.0)                  # input-dim units
    sk = pl.new_sketch()
    w = torch.zeros((64, 64), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(usk.UskError):
        usk.build_rows(pl, 0, 0, 32, w, sk)
    po = usk.plan_allocation([(64, 64)], bpw=2.0, granularity="outrow")
    so = po.new_sketch()
    with pytest.raises(usk.UskError):
        usk.build_rows(po, 0, 10, 70, w, so)                       # rows past out
    with pytest.raises(usk.UskError):
        usk.build_rows(po, 1, 0, 8, w, so)                         # layer out of range
