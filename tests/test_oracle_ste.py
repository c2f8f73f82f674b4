"""Pins of the aggregated-gradient baseline oracle (Figure 4a;
SPEC finetune module aggregated_backward) and its 2^-48 fixed-point definition (ledger)."""
import numpy as np

import synth

S48 = 2.0 ** 48


def fixed_sum(vals):
    return np.float32(float(np.sum(np.rint(np.asarray(vals, np.float64) * S48).astype(np.int64))) / S48)


def test_spec_example_shared_slot(orc):
    # two members with grads 0.1 and -0.3 sharing one slot -> -0.2 (SPEC aggregated_backward)
    # 2 fp32 weights at 16 bpw = 32 bits = one cell: both members share it
    pl1 = orc.plan([(2, 1)], 16.0, M=1, dtype=orc.F32, hash_kind=orc.HASH_IDENTITY)
    assert int(pl1.ncols[0]) == 1
    got = orc.aggregate_grad(pl1, 0, np.array([[0.1], [-0.3]]))
    assert got.tolist() == [fixed_sum([0.1, -0.3])]
    assert abs(float(got[0]) - (-0.2)) < 1e-7


def test_injective_mapping_is_identity(orc):
    # identity hash with N >= out: p mod N is injective inside a unit, one member per cell
    o, i = 16, 8
    pl = orc.plan([(o, i)], 64.0, M=1, dtype=orc.F32, hash_kind=orc.HASH_IDENTITY)
    assert (pl.ncols >= o).all()
    g = synth.weights_f32(o, i, 4).astype(np.float64)
    got = orc.aggregate_grad(pl, 0, g)
    for t in range(i):
        off = int(pl.offsets[t])
        for p in range(o):
            assert got[off + p] == np.float32(g[p, t])
        assert (got[off + o:off + int(pl.ncols[t])] == 0).all()  # empty cells


def test_matches_bucket_sums_and_fp64(orc):
    o, i, M = 64, 32, 3
    pl = orc.plan([(o, i)], 1.0, M=M, dtype=orc.BF16, seed=21)
    g = synth.weights_f32(o, i, 8).astype(np.float64) * 3.0
    got = orc.aggregate_grad(pl, 0, g)
    for t in range(i):
        N, off = int(pl.ncols[t]), int(pl.offsets[t])
        idx = orc.hash_indices(orc.HASH_X, 21, 0, t, M, np.arange(o), N)
        for r in range(M):
            for c in range(N):
                members = g[idx[r] == c, t]
                assert got[off + r * N + c] == fixed_sum(members)
                assert abs(float(got[off + r * N + c]) - members.sum()) <= len(members) * 2.0 ** -49 + \
                    abs(members.sum()) * 2.0 ** -23 + 1e-30


def test_finite_differences_shared_parameter(orc):
    # single-row aggregated mode (Figure 4a): w(p) = s[idx(p)], L(s) = sum_p c_p w(p)^2 / 2 + d_p w(p)
    # -> dL/ds[k] = sum over members of dL/dw(p), checked by central differences on s
    o, i = 8, 8
    pl = orc.plan([(o, i)], 8.0, M=1, dtype=orc.F32, seed=3)
    rng = np.random.default_rng(0)
    cpar = rng.uniform(0.5, 1.5, (o, i))
    dpar = rng.standard_normal((o, i))
    s = rng.standard_normal(int(pl.offsets[-1]))
    idx = np.zeros((o, i), dtype=np.int64)
    for t in range(i):
        idx[:, t] = pl.offsets[t] + orc.hash_indices(orc.HASH_X, 3, 0, t, 1, np.arange(o), int(pl.ncols[t]))[0]

    def loss(sv):
        w = sv[idx]
        return float(np.sum(cpar * w * w / 2 + dpar * w))

    gw = cpar * s[idx] + dpar  # dL/dw
    got = orc.aggregate_grad(pl, 0, gw)
    h = 1e-4
    for k in range(len(s)):
        e = np.zeros_like(s)
        e[k] = h
        fd = (loss(s + e) - loss(s - e)) / (2 * h)
        assert abs(float(got[k]) - fd) <= 1e-4 * max(1.0, abs(fd))
