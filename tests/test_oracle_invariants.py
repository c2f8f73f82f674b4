"""Invariants the paper states for AbsMaxMin, checked on the oracle at scale."""
import numpy as np
import pytest

import synth


@pytest.mark.parametrize("bpw", [16.0, 4.0])        # fp32 states: rate 1/2 and 1/8
@pytest.mark.parametrize("M", [1, 3])
def test_underestimate_1e6(orc, bpw, M):
    """|w'| <= |w| for every weight (PAPER.md:257-258 'either preserves the original value or
    represents it with a smaller absolute value').  10^6 weights."""
    out, inn = 1000, 1000
    W = synth.weights_f32(out, inn, seed=21)
    pl = orc.plan([(out, inn)], bpw, M=M, dtype=orc.F32, seed=77)
    sk = orc.build_model(pl, [W])
    Wr = orc.value_of(orc.reconstruct_rows(pl, sk, 0), orc.F32).reshape(out, inn)
    assert np.all(np.abs(Wr) <= np.abs(W.astype(np.float64)))
    # every reconstructed value is one of the layer's own weights (pure selection)
    assert np.isin(Wr.astype(np.float32), W).all()


def test_magnitude_monotone_in_rows(orc):
    """Rows are independent of M (DESIGN.md hash contract), so at fixed N adding a row can only
    raise |w'| towards |w|: the magnitude error |w| - |w'| never increases.
    SPEC's |w - w'| form does NOT hold when an opposite-signed collider wins (counterexample below,
    DESIGN.md L24)."""
    out, inn = 64, 200
    W = synth.weights_f32(out, inn, seed=5).astype(np.float64)
    prev = None
    for M in range(1, 6):
        pl = orc.plan([(out, inn)], 4.0 * M, M=M, dtype=orc.F32, seed=9)   # N fixed = out/8 per unit
        assert set(pl.ncols.tolist()) == {out // 8}
        sk = orc.build_model(pl, [W.astype(np.float32)])
        Wr = orc.value_of(orc.reconstruct_rows(pl, sk, 0), orc.F32).reshape(out, inn)
        mag_err = np.abs(W) - np.abs(Wr)
        if prev is not None:
            assert np.all(mag_err <= prev)
        prev = mag_err
    # counterexample to |w - w'| monotonicity: w = 0.5, row0 cell 0.4, row1 cell -0.45
    f = lambda v: int(np.array([v], np.float32).view(np.uint32)[0])
    one = orc.value_of([orc.retrieve(orc.F32, [f(0.4)])], orc.F32)[0]
    two = orc.value_of([orc.retrieve(orc.F32, [f(0.4), f(-0.45)])], orc.F32)[0]
    assert abs(0.5 - two) > abs(0.5 - one) and abs(0.5) - abs(two) < abs(0.5) - abs(one)


def test_determinism(orc):
    W = synth.weights_bf16(128, 96, seed=1)
    pl = orc.plan([(128, 96)], 0.5, M=3, dtype=orc.BF16, seed=1)
    a = orc.build_model(pl, [W])
    b = orc.build_model(pl, [W])
    assert a.tobytes() == b.tobytes()


def test_sign_errors_trace_to_colliders(orc):
    """Every sign error comes from an opposite-signed collider winning a bonded cell."""
    rng = np.random.default_rng(4)
    L, M, N = 4000, 3, 400
    w = rng.standard_normal(L).astype(np.float32)
    pos = np.arange(L, dtype=np.uint32)
    cells = orc.sketch_unit(w.view(np.uint32), pos, M, N, seed=3)
    rec = orc.value_of(orc.retrieve_unit(cells, pos, seed=3), orc.F32)
    idx = orc.hash_indices(orc.HASH_X, 3, 0, 0, M, pos, N)
    wrong = np.nonzero(np.sign(rec) != np.sign(w))[0]
    assert len(wrong) > 0
    for k in wrong:
        # the selected value is a weight of the unit with the opposite sign that shares a cell with k
        cands = [j for i in range(M) for j in np.nonzero(idx[i] == idx[i][k])[0] if j != k]
        assert any(np.float64(w[j]) == rec[k] and np.sign(w[j]) != np.sign(w[k]) for j in cands)
