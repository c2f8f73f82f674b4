"""Statistical pins: the oracle's collision statistics vs closed forms and the paper's numbers.

Under ideal random hashing a unit with k weights and N columns per row has bucket loads
Binomial(k, 1/N) (Appendix B), empty fraction (1 - 1/N)^k (Table 3), and
P(untouched) = int_0^1 1 - (1 - (1 - u/N)^(k-1))^M du for continuous weights (DESIGN.md
"Statistics").  A dropped row, a max/min swap, a wrong tie rule or a hash that is not
uniform fails these."""
import json
import math
import os

import numpy as np
import pytest
from scipy import integrate, stats

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))


def untouched_closed_form(k, N, M):
    f = lambda u: 1.0 - (1.0 - (1.0 - u / N) ** (k - 1)) ** M
    return integrate.quad(f, 0.0, 1.0, limit=200)[0]


def _unit(orc, k, N, M, seed, dist="normal"):
    rng = np.random.default_rng(seed)
    w = rng.standard_normal(k).astype(np.float32)
    pos = np.arange(k, dtype=np.uint32)
    cells = orc.sketch_unit(w.view(np.uint32), pos, M, N, seed=seed, layer=2, t=5)
    return w, pos, cells


def test_table3_unoccupied(orc):
    g = GOLD["table3_unoccupied"]
    k = 400_000
    for rate, paper_pct in zip(g["rates"], g["percent"]):
        N = int(k * rate)
        _, _, cells = _unit(orc, k, N, 1, seed=31)
        frac = float((cells == 0x7F800000).mean())
        expect = (1 - 1 / N) ** k
        sigma = math.sqrt(max(expect * (1 - expect), 1e-12) / N)
        assert abs(frac - expect) <= 4 * sigma + 1e-6, (rate, frac, expect)
        # the paper's printed value (Table 3) within half a percentage point
        assert abs(100 * frac - paper_pct) <= 0.5, (rate, 100 * frac, paper_pct)


@pytest.mark.parametrize("name", ["untouched_absmaxmin_rate_half", "untouched_sketch_rate_quarter"])
def test_untouched_vs_closed_form_and_paper(orc, name):
    g = GOLD[name]
    k, M = 120_000, g["rows"]
    N = int(round(k * g["rate"] / M))          # rate counts all M rows (L20)
    w, pos, cells = _unit(orc, k, N, M, seed=57)
    rec = orc.retrieve_unit(cells, pos, seed=57, layer=2, t=5)
    frac = float((rec == w.view(np.uint32)).mean())
    expect = untouched_closed_form(k, N, M)
    sigma = math.sqrt(expect * (1 - expect) / k)
    assert abs(frac - expect) <= 4 * sigma + 2e-3, (frac, expect)
    assert abs(100 * expect - g["percent"]) <= 0.1       # closed form vs the printed number
    assert abs(100 * frac - g["percent"]) <= 1.0         # measured vs the printed number


@pytest.mark.parametrize("M,lam", [(2, 64.0), (3, 96.0)])
def test_untouched_at_bench_loads(orc, M, lam):
    """Config 1 (M=2, lambda=64) and config 3 (M=3, lambda=96) loads: 2.34% / 1.91%."""
    k = 200_000
    N = int(k / lam)
    w, pos, cells = _unit(orc, k, N, M, seed=8)
    rec = orc.retrieve_unit(cells, pos, seed=8, layer=2, t=5)
    frac = float((rec == w.view(np.uint32)).mean())
    expect = untouched_closed_form(k, N, M)
    assert abs(frac - expect) <= 4 * math.sqrt(expect * (1 - expect) / k) + 1e-3


def test_bucket_loads_binomial(orc):
    """Per-row bucket loads ~ Binomial(k, 1/N) (Appendix B), chi-square over load classes."""
    k, N, M = 50_000, 5_000, 3
    idx = np.array([[orc.hash_index(0, 1234, 1, 7, i, p, N) for p in range(k)] for i in range(M)])
    for i in range(M):
        loads = np.bincount(idx[i], minlength=N)
        obs = np.bincount(np.minimum(loads, 20), minlength=21)
        pmf = stats.binom.pmf(np.arange(20), k, 1 / N)
        exp = np.append(pmf, 1 - pmf.sum()) * N
        keep = exp > 5
        chi2 = (((obs[keep] - exp[keep]) ** 2) / exp[keep]).sum()
        assert chi2 < stats.chi2.ppf(0.9999, keep.sum() - 1)
    # rows independent: pairs colliding in two rows ~ C(k,2)/N^2 per pair of rows
    for a, b in ((0, 1), (1, 2)):
        key = idx[a].astype(np.int64) * N + idx[b]
        cnt = np.bincount(key)
        pairs = int((cnt * (cnt - 1) // 2).sum())
        expect = k * (k - 1) / 2 / N**2
        assert abs(pairs - expect) <= 5 * math.sqrt(expect) + 2


@pytest.mark.parametrize("lam", [2, 4, 8])
@pytest.mark.parametrize("p", [0.5, 0.9, 0.99])
def test_eq6_error_bound(orc, lam, p):
    """Eq. 6 (proof PAPER.md:537-552, reading DESIGN.md L15): for an occupied
    bucket of load n holding s = the abs-min member, P(|s| >= F^-1_{|w|}(1 - p^{1/n})) = p for a
    continuous weight CDF; coverage must match p within 4 binomial standard errors."""
    k = 60_000
    N = k // lam
    w, pos, cells = _unit(orc, k, N, 1, seed=lam * 100 + int(p * 100))
    idx = np.array([orc.hash_index(0, lam * 100 + int(p * 100), 2, 5, 0, q, N) for q in range(k)])
    load = np.bincount(idx, minlength=N)
    occ = load > 0
    s = np.abs(orc.value_of(cells[0], orc.F32))[occ]
    n = load[occ]
    # |w| for w ~ N(0,1): F(x) = 2 Phi(x) - 1 => F^-1(q) = Phi^-1((1 + q) / 2)
    L = stats.norm.ppf((1.0 + (1.0 - p ** (1.0 / n))) / 2.0)
    cov = float((s >= L).mean())
    se = math.sqrt(p * (1 - p) / occ.sum())
    assert abs(cov - p) <= 4 * se + 1e-3, (cov, p)


def test_xg_layer_untouched_and_loads(orc):
    """USK-XG (L32) at the config-3 load: a ROW-unit layer (2048 positions per unit,
    M = 3, 0.5 bpw bf16 -> N = 21) sketched and reconstructed by the oracle.  Within each unit the
    family is the USK-X one, so the untouched fraction must still match Appendix B's closed form,
    and the per-row bucket loads of a group must be Binomial(k, 1/N); the 8 units of a key group
    share every index, different groups do not."""
    import oracle as O
    out, inn = 2048, 256
    pl = O.plan([(out, inn)], 0.5, M=3, dtype=O.BF16, hash_kind=O.HASH_XG, seed=41)
    N = int(pl.ncols[0])
    assert (np.asarray(pl.ncols) == N).all()
    rng = np.random.default_rng(41)
    W = (0.02 * rng.standard_normal((out, inn))).astype(np.float32)
    Wb = O.f32_to_bf16_rne(W.view(np.uint32)).astype(np.uint16)
    sk = O.build_model(pl, [Wb])
    rec = O.reconstruct_rows(pl, sk, 0)
    frac = float((rec == Wb).mean())
    expect = untouched_closed_form(out, N, 3)
    assert abs(frac - expect) <= 4 * math.sqrt(expect * (1 - expect) / (out * inn)) + 2e-3, (frac, expect)
    pos = np.arange(out, dtype=np.uint32)
    for g in range(0, inn // 8, 7):
        idx = O.hash_indices(O.HASH_XG, 41, 0, 8 * g, 3, pos, N)
        np.testing.assert_array_equal(idx, O.hash_indices(O.HASH_XG, 41, 0, 8 * g + 7, 3, pos, N))
        if g:
            assert (idx != O.hash_indices(O.HASH_XG, 41, 0, 0, 3, pos, N)).mean() > 0.8
        for i in range(3):
            loads = np.bincount(idx[i], minlength=N)
            chi2 = (((loads - out / N) ** 2) / (out / N)).sum()
            assert chi2 < stats.chi2.ppf(0.9999, N - 1)
