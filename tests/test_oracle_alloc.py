"""Allocation / plan properties (§3.4; SPEC.md:300-304 invariants)."""
import numpy as np
import pytest

import synth


def test_budget_conservation_random(orc):
    rng = np.random.default_rng(0)
    for _ in range(200):
        U = int(rng.integers(1, 300))
        C = int(rng.integers(1, min(U, 16) + 1))
        M = int(rng.integers(1, 4))
        mc = int(rng.integers(1, 4))
        scores = rng.exponential(size=U) * (rng.random(U) < 0.9)
        T = int(rng.integers(U * M * mc, U * M * 200))
        ncols, cls = orc.allocate(scores, T, C=C, M=M, min_cols=mc)
        used = int(M * ncols.sum())
        n_c = np.bincount(cls, minlength=C)
        assert used <= T
        assert used > T - max(n_c.max() * M, 1)            # largest-remainder leftover bound
        assert ncols.min() >= mc
        # classes are equal-count quantiles of the rank
        assert n_c.max() - n_c[n_c > 0].min() <= 1
        # one state size per class (per-class sketch regions)
        for c in range(C):
            assert len(set(ncols[cls == c].tolist())) <= 1


def test_monotonicity_per_unit(orc):
    """Raising one unit's score never decreases its allocation, C = U."""
    rng = np.random.default_rng(1)
    for _ in range(300):
        U = int(rng.integers(2, 40))
        s = rng.exponential(size=U) + 0.01
        T = int(rng.integers(U * 2, U * 100))
        a, _ = orc.allocate(s, T, min_cols=1)
        u = int(rng.integers(0, U))
        s2 = s.copy()
        s2[u] *= 1.0 + rng.exponential()
        b, _ = orc.allocate(s2, T, min_cols=1)
        assert b[u] >= a[u]


def test_scale_invariance(orc):
    """Power-of-two scalings are exact in the 2^24 fixed point => identical plans."""
    rng = np.random.default_rng(2)
    for _ in range(50):
        U = int(rng.integers(1, 200))
        s = rng.exponential(size=U)
        T = int(rng.integers(U * 3, U * 300))
        a = orc.allocate(s, T, C=4, M=3)
        for k in (0.25, 8.0, 2.0**40):
            b = orc.allocate(s * k, T, C=4, M=3)
            assert a[0].tolist() == b[0].tolist() and a[1].tolist() == b[1].tolist()


def test_plan_uniform_geometry_llama1b(orc):
    """Uniform importance, bf16 states, M=3, 0.5 bpw: per-unit columns follow floor(T / (U M))."""
    shapes = synth.llama_block(2048, 512, 8192)
    pl = orc.plan(shapes, 0.5, M=3, dtype=orc.BF16)
    want = {(2048, 2048): 21, (512, 2048): 5, (8192, 2048): 85, (2048, 8192): 21}
    for l, (o, i) in enumerate(shapes):
        u0, u1 = pl.layer_units(l)
        assert set(pl.ncols[u0:u1].tolist()) == {want[(o, i)]}
        T = (int(np.floor(0.5 * o * i))) // 16
        assert pl.acct[l, 2] == T
        assert pl.acct[l, 3] <= pl.acct[l, 0]
    assert pl.offsets[-1] == sum(3 * int(n) for n in pl.ncols)


def test_plan_classes_charge_map_bits(orc):
    """With C > 1 the 2-bit class map is charged against the per-layer budget (L9)."""
    s = [synth.saliency_like(2048, 1), synth.saliency_like(2048, 2), synth.saliency_like(8192, 3)]
    pl = orc.plan(synth.mlp_block_1b_shapes(), 0.5, M=3, dtype=orc.BF16, saliency=s, C=4)
    assert pl.acct[0, 1] == 2048 * 2 and pl.acct[2, 1] == 8192 * 2
    assert pl.acct[0, 2] == (int(0.5 * 8192 * 2048) - 4096) // 16 == 524032
    assert pl.acct[2, 2] == 523264
    for l in range(3):
        u0, u1 = pl.layer_units(l)
        assert pl.acct[l, 3] <= pl.acct[l, 0]
        # more salient classes never get fewer columns
        by_class = {int(c): int(n) for c, n in zip(pl.cls[u0:u1], pl.ncols[u0:u1])}
        cols = [by_class[c] for c in sorted(by_class)]
        assert cols == sorted(cols, reverse=True)


def test_plan_layer_granularity(orc):
    """LAYER: one unit per matrix, space proportional to mean importance x numel (L8)."""
    shapes = [(256, 256), (512, 256), (256, 512)]
    pl = orc.plan(shapes, 1.0, M=2, dtype=orc.F32, gran=orc.GRAN_LAYER, C=3,
                  saliency=[np.full(256, 1.0, np.float32), np.full(256, 1.0, np.float32),
                            np.full(512, 1.0, np.float32)])
    assert pl.unit_base.tolist() == [0, 1, 2, 3]
    T = sum(o * i for o, i in shapes) // 32
    assert 2 * pl.ncols.sum() <= T
    # equal mean importance -> columns proportional to numel: 1 : 2 : 2
    assert abs(pl.ncols[1] - 2 * pl.ncols[0]) <= 1 and abs(pl.ncols[2] - 2 * pl.ncols[0]) <= 1
    # config 1: 256x256 fp32, M=2, 1.0 bpw, LAYER -> T=2048, N=1024, exactly 1.0 bpw
    pl1 = orc.plan([(256, 256)], 1.0, M=2, dtype=orc.F32, gran=orc.GRAN_LAYER)
    assert pl1.ncols.tolist() == [1024] and pl1.acct[0, 3] == 256 * 256


def test_plan_errors(orc):
    with pytest.raises(orc.OracleError) as e:
        orc.plan([(512, 2048)], 0.5, M=3, dtype=orc.BF16, min_cols=16)   # 16 cells/unit < 3 x 16
    assert e.value.status == orc.EBUDGET
    with pytest.raises(orc.OracleError) as e:
        orc.plan([(64, 30)], 1.0, M=3, g=4)                                # g does not divide in
    assert e.value.status == orc.EINVAL
    with pytest.raises(orc.OracleError) as e:
        orc.plan([(64, 32)], 1.0, saliency=[np.full(32, -1.0, np.float32)])
    assert e.value.status == orc.EINVAL
    with pytest.raises(orc.OracleError) as e:
        orc.plan([(0, 32)], 1.0)
    assert e.value.status == orc.ESHAPE
