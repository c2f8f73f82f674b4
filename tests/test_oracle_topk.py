"""Pins of the Top-K outlier side table (Appendix A: "considers
weights with top-k large absolute values as important ones, stores them independently, and keeps
their value untouched"; ledger L29)."""
import numpy as np
import pytest

import synth


def test_topk_selection_matches_sort(orc):
    W = synth.weights_f32(40, 24, 3, scale=0.02)
    W[5, 7] = W[6, 8] = 0.5  # a tie: the smaller flat index ranks first
    W[9, 1] = -0.5
    idx, vals = orc.topk(orc.F32, W, 10)
    a = np.abs(W.ravel()).astype(np.float64)
    order = sorted(range(a.size), key=lambda e: (-a[e], e))[:10]
    assert idx.tolist() == sorted(order)
    np.testing.assert_array_equal(vals, W.ravel()[idx].view(np.uint32))
    idx2, _ = orc.topk(orc.F32, W, 2)
    assert idx2.tolist() == sorted([5 * 24 + 7, 6 * 24 + 8])  # |0.5| ties: flat index order


def test_outliers_excluded_from_the_sketch_and_exact(orc):
    o, i, M, K = 48, 32, 3, 30
    W = synth.weights_bf16(o, i, 6)
    pl = orc.plan([(o, i)], 4.0, M=M, dtype=orc.BF16, seed=12, topk=K)
    ts = orc.build_model(pl, [W])
    flat = set(ts.idx[0].tolist())
    assert len(flat) == K
    # cells == a sketch of the non-outlier weights only (direct per-unit sketch)
    for t in range(i):
        N, off = int(pl.ncols[t]), int(pl.offsets[t])
        keep = [p for p in range(o) if p * i + t not in flat]
        cells = orc.sketch_unit(W[keep, t].astype(np.uint32), np.array(keep), M, N, dtype=orc.BF16, seed=12,
                                t=t).ravel().astype(np.uint16)
        cells[cells == 0x7F80] = 0  # ledger L29: cells no remaining weight maps to hold +0, not +Inf
        np.testing.assert_array_equal(ts.cells[off:off + M * N], cells)
    Wp = orc.reconstruct_rows(pl, ts, 0)
    np.testing.assert_array_equal(Wp.ravel()[ts.idx[0]], ts.vals[0])  # untouched
    # linear over the overlaid W'
    x = synth.vector(i, seed=1)[0].astype(np.float64)
    np.testing.assert_allclose(orc.linear_rows(pl, ts, 0, x)[0], orc.value_of(Wp, orc.BF16) @ x, rtol=0, atol=1e-15)


def test_topk_accounting(orc):
    o, i, K = 64, 64, 100
    pl = orc.plan([(o, i)], 2.0, M=3, dtype=orc.BF16, topk=K)
    budget, meta, T, achieved = (int(x) for x in pl.acct[0])
    assert T == (budget - meta - K * (32 + 16)) // 16
    cells = int(pl.offsets[-1])
    assert achieved == cells * 16 + K * 48 + meta <= budget
    with pytest.raises(orc.OracleError):
        orc.plan([(o, i)], 2.0, M=3, dtype=orc.BF16, topk=o * i)  # side table > budget
    with pytest.raises(orc.OracleError):
        orc.plan([(o, i)], 2.0, M=3, dtype=orc.BF16, topk=K, gran=orc.GRAN_LAYER)


def test_topk_reduces_relative_error(orc):
    # App. A: "AbsMaxMin is an underestimate sketch, so removing values naturally reduces the
    # induced relative error" -- heavy-tailed weights, the SAME sketch cells with and without 1 %
    # outliers (the side table's bits are added to the budget): mean relative and absolute error
    # both drop, the outliers themselves are exact
    o, i = 512, 64
    rng = np.random.default_rng(5)
    W = synth.f32_to_bf16_bits((rng.standard_t(3, (o, i)) * 0.02).astype(np.float32))
    w = synth.bf16_bits_to_f32(W).astype(np.float64)
    nz = w != 0
    K = o * i // 100
    res = {}
    for k, bpw in ((0, 2.0), (K, 2.0 + K * 48 / (o * i))):
        pl = orc.plan([(o, i)], bpw, M=3, dtype=orc.BF16, seed=4, topk=k)
        Wp = orc.value_of(orc.reconstruct_rows(pl, orc.build_model(pl, [W]), 0), orc.BF16)
        res[k] = (int(pl.acct[0, 2]), np.mean(np.abs(w - Wp)[nz] / np.abs(w[nz])), np.mean(np.abs(w - Wp)))
    assert res[0][0] == res[K][0]  # equal sketch cells
    assert res[K][1] < res[0][1] and res[K][2] < res[0][2], res


def test_topk_sketch_values_finite_at_outliers(orc):
    # ledger L29: at 16 bpw a layer's cells outnumber its weights, so some cells receive only
    # outliers; they hold +0, and the sketch value w'_sketch at every outlier position (which the
    # GEMV correction x (w - w'_sketch) reads) is finite.  Without outliers no cell is +0-by-rule.
    o, i, M, K = 64, 64, 3, 64
    W = synth.weights_bf16(o, i, 9)
    pl = orc.plan([(o, i)], 16.0, M=M, dtype=orc.BF16, seed=3, topk=K)
    ts = orc.build_model(pl, [W])
    assert not np.any(ts.cells[:int(pl.offsets[-1])] == 0x7F80)  # no +Inf state left
    flat = ts.idx[0]
    for e in flat.tolist():
        oo, jj = divmod(e, i)
        N, off = int(pl.ncols[jj]), int(pl.offsets[jj])
        idx = orc.hash_indices(orc.HASH_X, 3, 0, jj, M, [oo], N)[:, 0]
        vals = [orc.value_of(np.array([ts.cells[off + r * N + int(c)]], np.uint16), orc.BF16)[0]
                for r, c in enumerate(idx)]
        assert all(np.isfinite(v) for v in vals)
    x = synth.vector(i, seed=2)[0].astype(np.float64)
    y = orc.linear_rows(pl, ts, 0, x)[0]
    assert np.all(np.isfinite(y))
