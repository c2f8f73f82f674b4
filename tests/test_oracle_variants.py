"""Pins of the comparison variants and the compression report (Appendix C.2,
PAPER.md:612-619; SPEC stats module and compare_variants; ledger L27)."""
import math

import numpy as np
import pytest

import synth

S48 = 2.0 ** 48


def _row_shapes(o, i):
    return [(o, i)]


def _build(orc, W, bpw, M, variant, dtype=None, hash_kind=None, seed=7):
    o, i = W.shape
    dtype = (orc.BF16 if W.dtype == np.uint16 else orc.F32) if dtype is None else dtype
    pl = orc.plan([(o, i)], bpw, M=M, dtype=dtype, seed=seed, variant=variant,
                  hash_kind=orc.HASH_X if hash_kind is None else hash_kind)
    sk = orc.build_model(pl, [W])
    return pl, sk, orc.reconstruct_rows(pl, sk, 0)


def test_absminmax_overestimates(orc):
    # AbsMaxMin underestimates |w|; swapping min and max gives |w'| >= |w|
    W = synth.weights_f32(64, 96, 3)
    pl, sk, Wp = _build(orc, W, 4.0, 3, orc.ABSMINMAX)
    assert (np.abs(Wp.view(np.float32)) >= np.abs(W)).all()
    # and cells start at +0: a cell nobody maps to holds +0
    occ = np.zeros(pl.total_cells, bool)
    for t in range(96):
        N, off = int(pl.ncols[t]), int(pl.offsets[t])
        idx = orc.hash_indices(orc.HASH_X, 7, 0, t, 3, np.arange(64), N)
        for r in range(3):
            occ[off + r * N + idx[r]] = True
    assert (sk.view(np.uint32)[~occ] == 0).all()


def test_countmin_single_row_is_bucket_sum(orc):
    # M = 1: w' = the sum of the weights in w's bucket (fixed point, rounded to the dtype)
    o, i = 48, 16
    W = synth.weights_f32(o, i, 5)
    pl, sk, Wp = _build(orc, W, 8.0, 1, orc.COUNTMIN)
    Wpf = Wp.view(np.float32)
    for t in range(i):
        N = int(pl.ncols[t])
        idx = orc.hash_indices(orc.HASH_X, 7, 0, t, 1, np.arange(o), N)[0]
        for p in range(o):
            members = W[idx == idx[p], t].astype(np.float64)
            want = np.float32(float(np.sum(np.rint(members * S48).astype(np.int64))) / S48)
            assert Wpf[p, t] == want
            assert abs(Wpf[p, t] - members.sum()) <= len(members) * 2.0 ** -49 + abs(members.sum()) * 2.0 ** -23


@pytest.mark.parametrize("variant", [0, 1, 2])
def test_injective_configs_are_exact(orc, variant):
    # SPEC compare_variants: identical injective configs -> all variants report zero error
    o, i = 32, 8
    W = synth.weights_f32(o, i, 9)
    pl, sk, Wp = _build(orc, W, 64.0, 1, variant, hash_kind=orc.HASH_IDENTITY)
    assert (pl.ncols >= o).all()
    np.testing.assert_array_equal(Wp.view(np.float32), W)
    st = orc.stats(pl, 0, W, Wp)
    assert st["untouched"] == st["weights"] == o * i and st["rel_exact"] == o * i
    assert st["sign_errors"] == 0


def test_stats_spec_examples(orc):
    # w = 0.5, w' = 0.4 -> relative error 0.2 (bin [0.1, 1)), no sign error;
    # w = 0.5, w' = -0.3 -> relative error 1.6 (bin [1, 10)), sign error; w = 0 counted apart
    pl = orc.plan([(4, 1)], 64.0, M=1, dtype=orc.F32, hash_kind=orc.HASH_IDENTITY)
    W = np.array([[0.5], [0.5], [0.0], [0.25]], np.float32)
    Wp = np.array([[0.4], [-0.3], [0.1], [0.25]], np.float32).view(np.uint32)
    st = orc.stats(pl, 0, W, Wp)
    assert st["weights"] == 4 and st["zero_weights"] == 1 and st["untouched"] == 1
    assert st["sign_errors"] == 1
    assert st["rel_1e-1"] == 1 and st["rel_1"] == 1 and st["rel_exact"] == 1
    assert st["cells"] == int(pl.ncols[0]) and st["unoccupied"] == int(pl.ncols[0]) - 4


def _mc(orc, variant, M, rate, seed):
    # single layer of Gaussian-like weights, ROW units of 2048 weights, M rows at `rate`
    o, i = 2048, 32
    W = synth.weights_f32(o, i, seed)
    bpw = 32.0 * rate
    pl, sk, Wp = _build(orc, W, bpw, M, variant, seed=seed)
    return pl, W, Wp, orc.stats(pl, 0, W, Wp)


def test_untouched_and_unoccupied_closed_forms(orc):
    # rate 1/2, M = 1 (lambda = 2, ledger L18): AbsMaxMin untouched = int_0^1 e^{-2u} du = 43.23 %
    # (paper 43.25 %); AbsMinMax equals it by u <-> 1-u symmetry; CountMin untouched = P(alone) =
    # e^{-2} = 13.53 % (paper 13.56 %); unoccupied = (1 - 1/m)^k ~ e^{-2} (Table 3: 13.53 %)
    n = 2048 * 32
    sd = lambda p: math.sqrt(p * (1 - p) / n)
    p_amm = (1 - math.exp(-2)) / 2
    for variant, p in ((0, p_amm), (1, p_amm), (2, math.exp(-2))):
        pl, W, Wp, st = _mc(orc, variant, 1, 0.5, 11)
        frac = st["untouched"] / st["weights"]
        assert abs(frac - p) <= 4 * sd(p) + 2e-3, (variant, frac, p)
        un = st["unoccupied"] / st["cells"]
        assert abs(un - math.exp(-2)) <= 4 * math.sqrt(math.exp(-2) / st["cells"]) + 2e-3, un


def test_variant_ordering(orc):
    # SPEC compare_variants (Figure 7 captions 1e0 / 1e6 / 1e7): at rate 1/2, mean relative error
    # AbsMaxMin < AbsMinMax < CountMin, and untouched fraction AbsMaxMin >= AbsMinMax > CountMin
    res = {}
    for variant in (0, 1, 2):
        pl, W, Wp, st = _mc(orc, variant, 3, 0.5, 12)
        w = W.astype(np.float64)
        wp = Wp.view(np.float32).astype(np.float64)
        nz = w != 0
        res[variant] = (np.mean(np.abs(w - wp)[nz] / np.abs(w[nz])), st["untouched"] / st["weights"])
    assert res[0][0] < res[1][0] < res[2][0], res
    assert res[0][1] >= res[1][1] - 0.01 and res[1][1] > res[2][1], res
