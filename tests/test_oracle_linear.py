"""Oracle linear / reconstruction vs independent references."""
import numpy as np
import pytest

import synth


@pytest.mark.parametrize("gran,g", [(0, 1), (0, 4), (1, 1)])
def test_linear_matches_numpy_fp64(orc, gran, g):
    """y = x W'^T in fp64: once W' is bit-checked, a library matmul is an independent
    reference."""
    out, inn = 96, 128
    W = synth.weights_bf16(out, inn, seed=3)
    pl = orc.plan([(out, inn)], 1.0, M=3, dtype=orc.BF16, gran=gran, g=g, seed=5)
    sk = orc.build_model(pl, [W])
    Wr = orc.value_of(orc.reconstruct_rows(pl, sk, 0), orc.BF16).reshape(out, inn)
    x = synth.vector(inn, seed=4, T=3).astype(np.float64)
    y = orc.linear_rows(pl, sk, 0, x)
    np.testing.assert_allclose(y, x @ Wr.T, rtol=1e-13, atol=1e-13)
    y2 = orc.linear_rows(pl, sk, 0, x, 10, 50)
    np.testing.assert_array_equal(y2, y[:, 10:50])


def test_reconstruct_entries_match_rows(orc):
    out, inn = 64, 80
    W = synth.weights_f32(out, inn, seed=1)
    pl = orc.plan([(out, inn)], 4.0, M=2, dtype=orc.F32, seed=8)
    sk = orc.build_model(pl, [W])
    full = orc.reconstruct_rows(pl, sk, 0)
    rng = np.random.default_rng(0)
    oj = np.stack([rng.integers(0, out, 100), rng.integers(0, inn, 100)], 1)
    np.testing.assert_array_equal(orc.reconstruct_entries(pl, sk, 0, oj), full[oj[:, 0], oj[:, 1]])


def test_partial_unit_build_matches_full(orc):
    """Building a unit range writes exactly the same cells as the full build (units independent,
    SPEC.md:118) -- the basis of layer/unit-sampled parity at full size."""
    out, inn = 128, 64
    W = synth.weights_bf16(out, inn, seed=2)
    pl = orc.plan([(out, inn)], 0.5, M=3, dtype=orc.BF16, seed=1)
    full = orc.build_model(pl, [W])
    part = np.zeros_like(full)
    orc.build_layer(pl, 0, W, part, 10, 20)
    o0, o1 = pl.offsets[10], pl.offsets[20]
    np.testing.assert_array_equal(part[o0:o1], full[o0:o1])
    assert not part[:o0].any() and not part[o1:].any()
