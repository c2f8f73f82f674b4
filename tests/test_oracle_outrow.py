"""Output-row units (SURVEY §8(f4) "Output-row units"; "each row of the weight matrix
corresponds to an independent AbsMaxMin sketch instance" read on PyTorch's [out, in] layout; ledger
L31): unit (l, o) holds the weights W[o, :] at positions p = j.

Pins: the sketch of W with output-row units IS the sketch of W^T with input-dim units (same unit
ids, positions and budgets), byte for byte, and W' transposes -- which ties this layout to the
already-pinned one; the set-based enumerator per unit; budget accounting; Appendix B's untouched
closed form at the unit load lambda = in / N; the error cases."""
import math

import numpy as np
import pytest
from scipy import integrate

import synth
from oracle import brute


@pytest.mark.parametrize("dtype", [0, 1])
@pytest.mark.parametrize("bpw", [2.0, 4.0])
def test_outrow_is_row_units_of_the_transpose(orc, dtype, bpw):
    shapes = [(96, 160), (40, 256)]
    Ws = [synth.weights_bf16(o, i, 70 + k) if dtype else synth.weights_f32(o, i, 70 + k) for k, (o, i) in
          enumerate(shapes)]
    a = orc.plan(shapes, bpw, M=3, dtype=dtype, gran=orc.GRAN_OUTROW, seed=12)
    b = orc.plan([(i, o) for o, i in shapes], bpw, M=3, dtype=dtype, gran=orc.GRAN_ROW, seed=12)
    for f in ("cls", "ncols", "offsets", "acct", "nrows", "unit_base"):
        np.testing.assert_array_equal(getattr(a, f), getattr(b, f))
    ska = orc.build_model(a, Ws)
    skb = orc.build_model(b, [np.ascontiguousarray(W.T) for W in Ws])
    np.testing.assert_array_equal(ska, skb)
    for l in range(len(shapes)):
        np.testing.assert_array_equal(orc.reconstruct_rows(a, ska, l), orc.reconstruct_rows(b, skb, l).T)


def test_outrow_brute_force(orc):
    out, inn = 20, 48
    pl = orc.plan([(out, inn)], 3.0, M=3, dtype=orc.F32, gran=orc.GRAN_OUTROW, seed=5)
    W = synth.edge_matrix_f32("mixed", out, inn, seed=2)
    sk = orc.build_model(pl, [W])
    Wp = orc.reconstruct_rows(pl, sk, 0)
    for o in range(out):
        M, N, off = int(pl.nrows[o]), int(pl.ncols[o]), int(pl.offsets[o])
        pos = np.arange(inn, dtype=np.uint32)                    # p = j
        idx = orc.hash_indices(orc.HASH_X, pl.seed, 0, o, M, pos, N)
        vals = W[o].astype(np.float64).tolist()
        S = brute.buckets(vals, idx, M, N)
        want = np.array([v for row in S for v in row], np.float32)
        np.testing.assert_array_equal(sk[off:off + M * N].view(np.float32), want)
        rec = np.array(brute.reconstruct(S, idx, M, inn), np.float32)
        np.testing.assert_array_equal(Wp[o].view(np.float32), rec)
    assert (np.abs(Wp.view(np.float32)) <= np.abs(W)).all()


def test_outrow_accounting(orc):
    shapes = [(300, 512), (128, 1024)]
    sal = [synth.saliency_like(512, 1), synth.saliency_like(1024, 2)]   # ignored within a layer (one class)
    pl = orc.plan(shapes, 0.5, M=3, dtype=orc.BF16, gran=orc.GRAN_OUTROW, saliency=sal, seed=3)
    assert pl.C == 1
    for l, (o, i) in enumerate(shapes):
        u0, u1 = pl.layer_units(l)
        assert u1 - u0 == o
        T = int(pl.acct[l, 2])
        assert T == (i * o // 2) // 16                             # floor(0.5 numel) / 16 bits
        N = T // (o * 3)
        assert (pl.ncols[u0:u1] == N).all()
        assert int(pl.acct[l, 3]) == o * 3 * N * 16 <= int(pl.acct[l, 0])


def test_outrow_untouched_closed_form(orc):
    out, inn = 3000, 512
    pl = orc.plan([(out, inn)], 2.0, M=3, dtype=orc.F32, gran=orc.GRAN_OUTROW, seed=9)
    W = synth.weights_f32(out, inn, seed=10)
    sk = orc.build_model(pl, [W])
    same = orc.reconstruct_rows(pl, sk, 0).view(np.uint32) == W.view(np.uint32)
    N = int(pl.ncols[0])
    f = lambda u: 1.0 - (1.0 - (1.0 - u / N) ** (inn - 1)) ** 3
    expect = integrate.quad(f, 0.0, 1.0, limit=200)[0]
    frac = float(same.mean())
    assert abs(frac - expect) <= 4 * math.sqrt(expect * (1 - expect) / same.size) + 2e-3, (frac, expect)


def test_outrow_errors(orc):
    for kw in ({"C": 2}, {"g": 2}):
        with pytest.raises(orc.OracleError) as e:
            orc.plan([(64, 64)], 1.0, M=3, gran=orc.GRAN_OUTROW, **kw)
        assert e.value.status == orc.EINVAL
