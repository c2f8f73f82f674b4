"""Per-class sketch rows (SURVEY §8(f4) "Per-class row counts M_c ('more rows')"; north star:
"importance-aware space allocation gives salient weights more rows or buckets"; categories
PAPER.md:523-528; DESIGN.md ledger L30).

Class c keeps M_c rows: its share of the layer's cells (still proportional to its importance,
x_c = T W_c / (W n_c M_c)) is split into M_c rows of N_c columns.  The pins below hold the oracle
to: a hand-worked allocation, the uniform plan when every M_c = M, cell conservation, the
set-based enumerator per unit, the underestimate invariant, the untouched closed form of
Appendix B per class (M_c rows at load lambda_c), and the error cases."""
import math

import numpy as np
import pytest
from scipy import integrate

import synth
from oracle import brute


def untouched_closed_form(k, N, M):
    f = lambda u: 1.0 - (1.0 - (1.0 - u / N) ** (k - 1)) ** M
    return integrate.quad(f, 0.0, 1.0, limit=200)[0]


def test_hand_worked_allocation(orc):
    """U = 8 units, scores 8,8,8,8,1,1,1,1 -> q = 2^24 (class 0) and 2^21 (class 1); T = 100,
    C = 2, M_c = (4, 1).  W_0 : W_1 = 8 : 1, so x_0 = 100 * 8/9 / (4 * 4) = 5.56 -> 5 and
    x_1 = 100 * 1/9 / (4 * 1) = 2.78 -> 2, using 80 + 8 = 88 cells; largest remainder
    (0.78 before 0.56): class 1 takes one column more for 4 cells (left 12 -> 8), class 0 would
    need 16 > 8.  N = (5, 3), 92 cells."""
    ncols, cls = orc.allocate([8, 8, 8, 8, 1, 1, 1, 1], 100, C=2, M=[4, 1])
    np.testing.assert_array_equal(cls, [0, 0, 0, 0, 1, 1, 1, 1])
    np.testing.assert_array_equal(ncols, [5, 5, 5, 5, 3, 3, 3, 3])
    # the same with one row count for both classes (M = 1): x = 88.9 / 4 = 22.2, 11.1 / 4 = 2.78
    ncols1, _ = orc.allocate([8, 8, 8, 8, 1, 1, 1, 1], 100, C=2, M=1)
    np.testing.assert_array_equal(ncols1, [22, 22, 22, 22, 3, 3, 3, 3])


def test_uniform_rows_reduce_to_the_plain_plan(orc):
    shapes = [(96, 64), (64, 128)]
    sal = [synth.saliency_like(64, seed=3), synth.saliency_like(128, seed=4)]
    a = orc.plan(shapes, 1.5, M=3, dtype=orc.BF16, saliency=sal, C=4, seed=9)
    b = orc.plan(shapes, 1.5, M=3, dtype=orc.BF16, saliency=sal, C=4, seed=9, class_rows=[3, 3, 3, 3])
    for f in ("cls", "ncols", "offsets", "acct", "nrows", "unit_base"):
        np.testing.assert_array_equal(getattr(a, f), getattr(b, f))
    assert (a.nrows == 3).all()


@pytest.mark.parametrize("state_bits", [0, 4])
def test_conservation_and_accounting(orc, state_bits):
    shapes = [(256, 192), (128, 256)]
    sal = [synth.saliency_like(192, seed=11), synth.saliency_like(256, seed=12)]
    rows = [4, 3, 2, 1]
    pl = orc.plan(shapes, 0.6, M=4, dtype=orc.BF16, saliency=sal, C=4, seed=5, class_rows=rows,
                  state_bits=state_bits)
    for l in range(len(shapes)):
        u0, u1 = pl.layer_units(l)
        cls, ncols, nrows = pl.cls[u0:u1], pl.ncols[u0:u1], pl.nrows[u0:u1]
        np.testing.assert_array_equal(nrows, np.array(rows)[cls])
        ends = pl.offsets[u0:u1] + nrows.astype(np.int64) * ncols
        np.testing.assert_array_equal(pl.offsets[u0 + 1:u1], ends[:-1])
        assert pl.offsets[u1] >= ends[-1]                      # (quantised: next layer G-aligned)
        cells = int((nrows.astype(np.int64) * ncols).sum())
        T = int(pl.acct[l, 2])
        n_c = np.bincount(cls, minlength=4)
        assert cells <= T
        assert T - cells < max(int(n_c[c]) * rows[c] for c in range(4) if n_c[c])  # largest remainder
        # more salient classes get at least as many cells per unit (q-ordered classes)
        per_unit = [int(rows[c] * ncols[cls == c][0]) for c in range(4) if n_c[c]]
        assert per_unit == sorted(per_unit, reverse=True)
        budget, meta, _, achieved = (int(v) for v in pl.acct[l])
        assert achieved <= budget
        if state_bits == 0:
            assert achieved == cells * 16 + meta


@pytest.mark.parametrize("dtype", [0, 1])
def test_brute_force_per_unit_rows(orc, dtype):
    """Bucket contents and W' of every unit (own M_u) vs the set-based enumerator."""
    out, inn = 48, 12
    sal = np.linspace(4.0, 0.5, inn).astype(np.float32)
    pl = orc.plan([(out, inn)], 2.0 if dtype == 1 else 4.0, M=3, dtype=dtype, saliency=[sal], C=3,
                  class_rows=[3, 2, 1], seed=21)
    assert set(pl.nrows.tolist()) == {1, 2, 3}
    W = synth.edge_matrix_bf16("mixed", out, inn, seed=4) if dtype == 1 else \
        synth.edge_matrix_f32("mixed", out, inn, seed=4)
    sk = orc.build_model(pl, [W])
    Wp = orc.reconstruct_rows(pl, sk, 0)
    bits = W.astype(np.uint32) if dtype == 1 else W.view(np.uint32)
    for t in range(inn):
        M, N, off = int(pl.nrows[t]), int(pl.ncols[t]), int(pl.offsets[t])
        pos = np.arange(out, dtype=np.uint32)                  # g = 1: p = o
        vals = orc.value_of(bits[:, t], dtype).tolist()
        idx = orc.hash_indices(orc.HASH_X, pl.seed, 0, t, M, pos, N)
        S = brute.buckets(vals, idx, M, N)
        inf = 0x7F80 if dtype else 0x7F800000
        want = [inf if math.isinf(v) else int(orc.bits_of(np.array([v], np.float32), 0)[0]) >> (16 if dtype else 0)
                for row in S for v in row]
        np.testing.assert_array_equal(sk[off:off + M * N].astype(np.uint32), np.array(want, np.uint32))
        rec = brute.reconstruct(S, idx, M, out)
        want_r = [int(orc.bits_of(np.array([v], np.float32), 0)[0]) >> (16 if dtype else 0) for v in rec]
        np.testing.assert_array_equal(Wp[:, t].astype(np.uint32), np.array(want_r, np.uint32))
    # the underestimate invariant on every weight
    assert (np.abs(orc.value_of(Wp, dtype)) <= np.abs(orc.value_of(bits, dtype))).all()


def test_untouched_per_class_closed_form(orc):
    """Two classes of units, M_c = (3, 1): each class's untouched fraction follows Appendix B's
    closed form at its own (k, N_c, M_c).  (At equal cells per unit and this load, lambda = 96
    vs 32, the 3-row class keeps FEWER weights exactly, 1.9 % vs 3.1 %: rows trade columns,
    PAPER.md:255 "the number of rows and columns of sketch state is a trade-off".)"""
    out, inn = 6000, 32
    sal = np.where(np.arange(inn) < 16, 1.0, 0.999).astype(np.float32)
    pl = orc.plan([(out, inn)], 1.0, M=3, dtype=orc.F32, saliency=[sal], C=2, class_rows=[3, 1], seed=77)
    W = synth.weights_f32(out, inn, seed=78)
    sk = orc.build_model(pl, [W])
    Wp = orc.reconstruct_rows(pl, sk, 0)
    same = (Wp.view(np.uint32) == W.view(np.uint32))
    fr = []
    for c, M in ((0, 3), (1, 1)):
        units = np.nonzero(pl.cls == c)[0]
        assert (pl.nrows[units] == M).all()
        N = int(pl.ncols[units[0]])
        frac = float(same[:, units].mean())
        expect = untouched_closed_form(out, N, M)
        sigma = math.sqrt(expect * (1 - expect) / (out * len(units)))
        assert abs(frac - expect) <= 4 * sigma + 2e-3, (c, frac, expect)
        fr.append(frac)
    assert fr[0] < fr[1]


def test_layer_granularity_per_class_rows(orc):
    """LAYER units: each layer is one unit of its class's rows; accounting and brute W'."""
    shapes = [(32, 16), (16, 32), (24, 8)]
    sal = [np.full(16, 4.0, np.float32), np.full(32, 1.0, np.float32), np.full(8, 0.25, np.float32)]
    pl = orc.plan(shapes, 1.0, M=3, dtype=orc.F32, saliency=sal, gran=orc.GRAN_LAYER, C=3, class_rows=[3, 2, 1],
                  seed=3)
    np.testing.assert_array_equal(pl.nrows, [3, 2, 1])
    np.testing.assert_array_equal(np.diff(pl.offsets), pl.nrows.astype(np.int64) * pl.ncols)
    Ws = [synth.weights_f32(o, i, seed=40 + l) for l, (o, i) in enumerate(shapes)]
    sk = orc.build_model(pl, Ws)
    for l, (o, i) in enumerate(shapes):
        Wp = orc.reconstruct_rows(pl, sk, l)
        M, N, off = int(pl.nrows[l]), int(pl.ncols[l]), int(pl.offsets[l])
        pos = np.array([j * o + r for r in range(o) for j in range(i)], np.uint32)   # p = j * out + o
        vals = Ws[l].astype(np.float64).ravel().tolist()
        idx = orc.hash_indices(orc.HASH_X, pl.seed, l, 0, M, pos, N)
        S = brute.buckets(vals, idx, M, N)
        rec = np.array(brute.reconstruct(S, idx, M, len(vals)), np.float32).reshape(o, i)
        np.testing.assert_array_equal(Wp.view(np.uint32), rec.view(np.uint32))


def test_errors(orc):
    shapes = [(32, 32)]
    with pytest.raises(orc.OracleError) as e:
        orc.plan(shapes, 1.0, M=3, C=2, class_rows=[3])             # one count per class
    assert e.value.status == orc.EINVAL
    for bad in ([0, 1], [9, 1]):
        with pytest.raises(orc.OracleError) as e:
            orc.plan(shapes, 1.0, M=3, C=2, class_rows=bad)
        assert e.value.status == orc.EINVAL
    with pytest.raises(orc.OracleError) as e:
        orc.plan(shapes, 1.0, M=3, C=2, class_rows=[3, 1], layer_importance=[1.0])
    assert e.value.status == orc.EINVAL
    with pytest.raises(orc.OracleError) as e:                        # floors sum_c n_c M_c min_cols > T
        orc.plan(shapes, 0.05, M=3, C=2, class_rows=[8, 8], min_cols=2)
    assert e.value.status == orc.EBUDGET
