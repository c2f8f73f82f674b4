"""Oracle pins for importance classes under USK-XG keys (DESIGN.md ledger L33): a ROW unit of an XG
plan scores by the mean saliency of its key group (8 consecutive units, the group that shares the
unit key, L32), so the 8 units of a group land in one class with one column count.

The grouping is checked against scores computed here by plain Python (sequential fp64 sums of the
group's saliency, §3.4 "importance-aware" scores), fed to the oracle's allocator (pinned by
tests/test_oracle_alloc*.py), and against invariants: groups uniform, higher-scored groups never get
fewer columns, USK-X plans keep per-unit scores, uniform saliency makes XG and X plans identical."""
import numpy as np
import pytest

import synth

CASES = [
    ([(256, 512), (128, 256)], None),
    ([(2048, 2048), (512, 2048), (8192, 512)], (3, 3, 2, 2)),
    ([(960, 72), (640, 40)], None),  # 9 and 5 key groups: class boundaries fall inside groups
]


def group_scores(sal, g_units=8):
    """Per-unit score = the sequential fp64 mean of the saliency of the unit's key group."""
    U = len(sal)
    out = np.zeros(U)
    for t in range(U):
        t0 = t // g_units * g_units
        t1 = min(t0 + g_units, U)
        s = 0.0
        for j in range(t0, t1):
            s += float(sal[j])
        out[t] = s / (t1 - t0)
    return out


@pytest.mark.parametrize("case", range(len(CASES)))
def test_xg_classes_follow_group_scores(orc, case):
    O = orc
    shapes, crows = CASES[case]
    sal = [synth.saliency_like(i, 300 + k) for k, (o, i) in enumerate(shapes)]
    pl = O.plan(shapes, 0.5, M=3, dtype=O.BF16, hash_kind=O.HASH_XG, seed=3, saliency=sal, C=4, class_rows=crows)
    for l, (o, i) in enumerate(shapes):
        u0, u1 = pl.layer_units(l)
        s = group_scores(sal[l])
        ncols, cls = O.allocate(s, int(pl.acct[l, 2]), C=4, M=3 if crows is None else crows)
        np.testing.assert_array_equal(pl.cls[u0:u1], cls)
        np.testing.assert_array_equal(pl.ncols[u0:u1], ncols)
        if crows is not None:
            np.testing.assert_array_equal(pl.nrows[u0:u1], np.asarray(crows)[cls])
        # groups uniform whenever the layer's class sizes are multiples of 8 units (in % 32 == 0)
        if i % 32 == 0:
            for a in (pl.cls[u0:u1], pl.ncols[u0:u1], pl.nrows[u0:u1]):
                assert (a.reshape(-1, 8) == a.reshape(-1, 8)[:, :1]).all()
        # a group scored higher never gets a lower class, nor (equal class rows) fewer columns
        order = np.argsort(-s, kind="stable")
        assert (np.diff(pl.cls[u0:u1][order].astype(int)) >= 0).all()
        if crows is None:
            assert (np.diff(pl.ncols[u0:u1][order]) <= 0).all()


def test_x_keeps_unit_scores_and_uniform_saliency_agrees(orc):
    O = orc
    shapes = [(256, 512), (128, 256)]
    sal = [synth.saliency_like(i, 310 + k) for k, (o, i) in enumerate(shapes)]
    px = O.plan(shapes, 0.5, M=3, dtype=O.BF16, hash_kind=O.HASH_X, seed=3, saliency=sal, C=4)
    for l, (o, i) in enumerate(shapes):
        u0, u1 = px.layer_units(l)
        ncols, cls = O.allocate(np.asarray(sal[l], dtype=np.float64), int(px.acct[l, 2]), C=4, M=3)
        np.testing.assert_array_equal(px.cls[u0:u1], cls)
        np.testing.assert_array_equal(px.ncols[u0:u1], ncols)
    # the per-unit X plan splits some group (the saliency is not constant over groups) ...
    assert any((px.cls[u0:u1].reshape(-1, 8) != px.cls[u0:u1].reshape(-1, 8)[:, :1]).any()
               for u0, u1 in (px.layer_units(l) for l in range(len(shapes))))
    # ... and with uniform saliency the grouping changes nothing
    flat = [np.ones(i, np.float32) for (o, i) in shapes]
    a = O.plan(shapes, 0.5, M=3, dtype=O.BF16, hash_kind=O.HASH_XG, seed=3, saliency=flat, C=4)
    b = O.plan(shapes, 0.5, M=3, dtype=O.BF16, hash_kind=O.HASH_X, seed=3, saliency=flat, C=4)
    np.testing.assert_array_equal(a.cls, b.cls)
    np.testing.assert_array_equal(a.ncols, b.ncols)
    np.testing.assert_array_equal(a.offsets, b.offsets)
