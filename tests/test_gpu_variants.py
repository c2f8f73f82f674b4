"""GPU parity of the comparison variants and the compression report (Appendix C.2,
PAPER.md:612-619; ledger L27): AbsMinMax / CountMin sketches and reconstructions bit-exact
against the oracle, sketch-GEMV within the 1e-5 bar, usk_stats counts equal to the oracle's."""
import numpy as np
import pytest

import synth
from test_gpu_parity import DT, assert_plan_equal, make_weights, sketch_cells, to_dev, w_bits

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

VAR = {"absmaxmin": 0, "absminmax": 1, "countmin": 2}


@pytest.fixture(scope="module")
def usk():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2506_17255_b200 import usk as u
    return u


CASES = [
    # (shapes, dtype, bpw, M, gran, g, hash, variant)
    ([(96, 64), (40, 96)], "bf16", 2.0, 3, "row", 1, "x", "absminmax"),
    ([(96, 64), (40, 96)], "bf16", 2.0, 3, "row", 1, "x", "countmin"),
    ([(256, 64)], "f32", 2.0, 2, "row", 1, "x", "absminmax"),
    ([(256, 64)], "f32", 2.0, 2, "row", 1, "x", "countmin"),
    ([(130, 64)], "bf16", 2.0, 3, "row", 2, "x", "countmin"),
    ([(96, 64), (64, 32)], "bf16", 2.0, 3, "layer", 1, "x", "absminmax"),
    ([(70, 64)], "f32", 8.0, 1, "row", 1, "identity", "countmin"),
]


@pytest.mark.parametrize("case", CASES, ids=[f"{c[7]}-{c[1]}-{c[4]}-g{c[5]}-M{c[3]}-{c[6]}" for c in CASES])
def test_variant_build_reconstruct_gemv_stats(orc, usk, case):
    shapes, dtype, bpw, M, gran, g, hk, var = case
    Ws = make_weights(shapes, dtype, 13)
    pl = usk.plan_allocation(shapes, bpw=bpw, rows=M, granularity=gran, dims_per_unit=g, hash=hk, dtype=dtype,
                             seed=77, variant=var)
    opl = orc.plan(shapes, bpw, M=M, dtype=DT[dtype], gran=1 if gran == "layer" else 0, g=g,
                   hash_kind=0 if hk == "x" else 1, seed=77, variant=VAR[var])
    assert_plan_equal(pl, opl)
    sk = pl.new_sketch()
    sk.fill_(0x5A)
    dW = [to_dev(W, dtype) for W in Ws]
    usk.build(pl, dW, sk)
    usk.check(pl)
    osk = orc.build_model(opl, Ws)
    np.testing.assert_array_equal(sketch_cells(sk, pl, dtype), osk)
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    for l, (o, i) in enumerate(shapes):
        Wr = torch.empty((o, i), dtype=tdt, device="cuda")
        usk.reconstruct(pl, sk, l, Wr)
        want = orc.reconstruct_rows(opl, osk, l)
        np.testing.assert_array_equal(w_bits(Wr, dtype), want)
        # GEMV against the oracle's fp64 product with the reconstructed weights
        xv = synth.vector(i, seed=5 + l)[0]
        x = torch.from_numpy(xv.astype(np.float32)).cuda()
        y = torch.empty(o, dtype=torch.float32, device="cuda")
        usk.linear(pl, sk, l, x.view(1, -1), y.view(1, -1), usk.new_workspace(pl, l))
        Wv = orc.value_of(want, DT[dtype])
        y64 = orc.linear_rows(opl, osk, l, xv.astype(np.float64))[0]
        denom = np.abs(Wv) @ np.abs(xv.astype(np.float64))
        err = np.abs(y.cpu().numpy().astype(np.float64) - y64) / np.maximum(denom, 1e-30)
        assert err.max() <= 1e-5, err.max()
        # the compression report
        got = usk.stats(pl, sk, l, dW[l])
        ref = orc.stats(opl, l, Ws[l], want)
        assert got == ref, (got, ref)


def test_stats_default_sketch_and_quantised(orc, usk):
    # usk_stats on the paper's sketch (raw bf16) and on a q4 plan equals the oracle's report
    shapes = [(128, 96)]
    W = synth.weights_bf16(128, 96, 3)
    for q in (0, 4):
        pl = usk.plan_allocation(shapes, bpw=2.0, rows=3, dtype="bf16", seed=8, state_bits=q, group_size=64 if q else 0)
        opl = orc.plan(shapes, 2.0, M=3, dtype=orc.BF16, seed=8, state_bits=q, group=64)
        sk = pl.new_sketch()
        dW = to_dev(W, "bf16")
        usk.build(pl, [dW], sk)
        osk = orc.build_model(opl, [W])
        got = usk.stats(pl, sk, 0, dW)
        ref = orc.stats(opl, 0, W, orc.reconstruct_rows(opl, osk, 0))
        assert got == ref, (q, got, ref)
        if q == 0:  # the AbsMaxMin underestimate: no weight grows, so no relative error >= 1 from growth
            assert got["untouched"] > 0
