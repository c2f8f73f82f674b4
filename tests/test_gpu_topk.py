"""GPU parity of the Top-K outlier side table (Appendix A; ledger
L29): plan accounting, the device top-K selection (side table bytes), the sketch of the remaining
weights, reconstructions with the overlay bit-exact; GEMV within the 1e-5 bar; bf16 prefill."""
import numpy as np
import pytest

import synth
from test_gpu_parity import DT, assert_plan_equal, make_weights, sketch_cells, to_dev, w_bits

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def usk():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2506_17255_b200 import usk as u
    return u


def side_table(sk, pl, l, dtype):
    li = pl.layers[l]
    a = sk.cpu().numpy()
    K = li.n_outliers
    idx = a[li.outlier_offset:li.outlier_offset + 4 * K].view(np.int32)
    v0 = li.outlier_offset + (4 * K + 15) // 16 * 16
    vals = a[v0:v0 + K * (2 if dtype == "bf16" else 4)].view(np.uint16 if dtype == "bf16" else np.uint32)
    return idx, vals


CASES = [
    # (shapes, dtype, bpw, M, g, topk)
    ([(256, 128), (96, 64)], "bf16", 2.0, 3, 1, 40),
    ([(300, 96)], "f32", 4.0, 2, 1, 100),
    ([(130, 64)], "bf16", 3.0, 3, 2, 25),       # dims_per_unit = 2: generic paths
    ([(64, 256)], "bf16", 4.0, 5, 1, 64),       # runtime-M kernel
]


@pytest.mark.parametrize("case", CASES, ids=[f"{c[1]}-g{c[4]}-M{c[3]}-K{c[5]}" for c in CASES])
def test_topk_parity(orc, usk, case):
    shapes, dtype, bpw, M, g, K = case
    Ws = make_weights(shapes, dtype, 21)
    pl = usk.plan_allocation(shapes, bpw=bpw, rows=M, dims_per_unit=g, dtype=dtype, seed=61, topk=K)
    opl = orc.plan(shapes, bpw, M=M, dtype=DT[dtype], g=g, seed=61, topk=K)
    assert_plan_equal(pl, opl)
    sk = pl.new_sketch()
    sk.fill_(0x3C)
    dW = [to_dev(W, dtype) for W in Ws]
    usk.build(pl, dW, sk)
    usk.check(pl)
    ts = orc.build_model(opl, Ws)
    np.testing.assert_array_equal(sketch_cells(sk, pl, dtype), ts.cells)
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    for l, (o, i) in enumerate(shapes):
        idx, vals = side_table(sk, pl, l, dtype)
        np.testing.assert_array_equal(idx.astype(np.int64), ts.idx[l])
        np.testing.assert_array_equal(vals.astype(np.uint32), ts.vals[l].astype(np.uint32))
        Wr = torch.empty((o, i), dtype=tdt, device="cuda")
        usk.reconstruct(pl, sk, l, Wr)
        want = orc.reconstruct_rows(opl, ts, l)
        np.testing.assert_array_equal(w_bits(Wr, dtype), want)
        r0, r1 = o // 4, o // 4 + 9
        buf = torch.zeros((r1 - r0, i + 8), dtype=tdt, device="cuda")
        usk.reconstruct(pl, sk, l, buf[:, :i], r0, r1)
        np.testing.assert_array_equal(w_bits(buf[:, :i].contiguous(), dtype), want[r0:r1])
        xv = synth.vector(i, seed=9 + l)[0]
        x = torch.from_numpy(xv.astype(np.float32)).cuda()
        y = torch.empty(o, dtype=torch.float32, device="cuda")
        usk.linear(pl, sk, l, x.view(1, -1), y.view(1, -1), usk.new_workspace(pl, l))
        Wv = orc.value_of(want, DT[dtype])
        y64 = Wv @ xv.astype(np.float64)
        err = np.abs(y.cpu().numpy().astype(np.float64) - y64) / np.maximum(np.abs(Wv) @ np.abs(xv.astype(np.float64)),
                                                                              1e-30)
        assert err.max() <= 1e-5, err.max()
        # output-sharded range (decode on several GPUs)
        ya = torch.empty(r1 - r0, dtype=torch.float32, device="cuda")
        usk.linear(pl, sk, l, x.view(1, -1), ya.view(1, -1), usk.new_workspace(pl, l, 1, r0, r1), r0, r1)
        np.testing.assert_array_equal(ya.cpu().numpy(), y.cpu().numpy()[r0:r1])
        st = usk.stats(pl, sk, l, dW[l])
        assert st == orc.stats(opl, l, Ws[l], want)


def test_topk_prefill(orc, usk):
    shapes = [(256, 128)]
    Ws = make_weights(shapes, "bf16", 4)
    pl = usk.plan_allocation(shapes, bpw=2.0, rows=3, dtype="bf16", seed=2, topk=50)
    opl = orc.plan(shapes, 2.0, M=3, dtype=orc.BF16, seed=2, topk=50)
    sk = pl.new_sketch()
    usk.build(pl, [to_dev(Ws[0], "bf16")], sk)
    ts = orc.build_model(opl, Ws)
    T = 80
    Xb = synth.f32_to_bf16_bits(synth.vector(128, seed=3, T=T).astype(np.float32))
    x = torch.from_numpy(Xb.view(np.int16).copy()).view(torch.bfloat16).cuda()
    y = torch.empty((T, 256), dtype=torch.bfloat16, device="cuda")
    usk.linear(pl, sk, 0, x, y, usk.new_workspace(pl, 0, T))
    ref = synth.bf16_bits_to_f32(Xb).astype(np.float64) @ orc.value_of(orc.reconstruct_rows(opl, ts, 0), orc.BF16).T
    rel = np.abs(y.float().cpu().numpy() - ref).max() / np.abs(ref).max()
    assert rel <= 2e-2, rel


def test_topk_full_layer_selection(orc, usk):
    # Llama-3.2-1B gate shape at 0.5 bpw with 64 outliers: the device top-K over 16.8 M weights equals
    # the oracle's exact selection
    o, i = 8192, 2048
    W = synth.weights_bf16(o, i, synth.seed_for(2, 0, 4))
    pl = usk.plan_allocation([(o, i)], bpw=0.5, rows=3, dtype="bf16", seed=0x5EED, topk=64)
    sk = pl.new_sketch()
    usk.build(pl, [to_dev(W, "bf16")], sk)
    usk.check(pl)
    idx, vals = side_table(sk, pl, 0, "bf16")
    want_idx, want_vals = orc.topk(orc.BF16, W, 64)
    np.testing.assert_array_equal(idx.astype(np.int64), want_idx)
    np.testing.assert_array_equal(vals.astype(np.uint32), want_vals)


@pytest.mark.parametrize("bpw,g", [(8.0, 1), (12.0, 1), (16.0, 1), (16.0, 2)])
def test_topk_high_bpw_finite(orc, usk, bpw, g):
    # ledger L29 (round 2): at 8-16 bpw some cells receive only outliers; they hold +0, so the GEMV's
    # outlier correction x (w - w'_sketch) stays finite (an +Inf state gave Inf - Inf = NaN)
    o, i, K = 512, 256, 96
    Ws = make_weights([(o, i)], "bf16", 31)
    pl = usk.plan_allocation([(o, i)], bpw=bpw, rows=3, dims_per_unit=g, dtype="bf16", seed=77, topk=K)
    opl = orc.plan([(o, i)], bpw, M=3, dtype=orc.BF16, g=g, seed=77, topk=K)
    sk = pl.new_sketch()
    usk.build(pl, [to_dev(Ws[0], "bf16")], sk)
    usk.check(pl)
    ts = orc.build_model(opl, Ws)
    np.testing.assert_array_equal(sketch_cells(sk, pl, "bf16"), ts.cells)
    assert not np.any(ts.cells == 0x7F80)
    want = orc.reconstruct_rows(opl, ts, 0)
    Wv = orc.value_of(want, orc.BF16)
    for xdt in ("f32", "bf16"):
        xv = synth.vector(i, seed=5)[0]
        if xdt == "bf16":
            xb = synth.f32_to_bf16_bits(xv)
            x = torch.from_numpy(xb.view(np.int16).copy()).view(torch.bfloat16).cuda()
            xv = synth.bf16_bits_to_f32(xb)
        else:
            x = torch.from_numpy(xv.astype(np.float32)).cuda()
        y = torch.empty(o, dtype=torch.float32, device="cuda")
        usk.linear(pl, sk, 0, x.view(1, -1), y.view(1, -1), usk.new_workspace(pl, 0))
        yh = y.cpu().numpy().astype(np.float64)
        assert np.all(np.isfinite(yh))
        x64 = xv.astype(np.float64)
        err = np.abs(yh - Wv @ x64) / np.maximum(np.abs(Wv) @ np.abs(x64), 1e-30)
        assert err.max() <= 1e-5, (xdt, err.max())
