"""Oracle (streaming Eq. 4 updates, usk_oracle.c) vs the set-based enumerator (oracle/brute.py)
on tiny inputs covering +-x ties, +-0, subnormals, every M <= 3 and N <= 8, both hash kinds,
and random insertion orders (SPEC.md:103 order independence)."""
import math

import numpy as np
import pytest

from oracle import brute
import synth


def _values_f32(rng, L):
    pool = np.array([0.5, -0.5, 0.25, -0.25, 0.0, -0.0, 1e-40, -1e-40, 3.0, -3.0, 0.125], np.float32)
    w = rng.standard_normal(L).astype(np.float32)
    pick = rng.random(L) < 0.6
    w[pick] = rng.choice(pool, size=int(pick.sum()))
    return w


def _to_bits(vals, dtype):
    a = np.array(vals, dtype=np.float32)
    b = a.view(np.uint32)
    return (b >> np.uint32(16)) if dtype == 1 else b


@pytest.mark.parametrize("dtype", [0, 1])
@pytest.mark.parametrize("hash_kind", [0, 1, 2])
def test_brute_force_buckets_and_reconstruction(orc, dtype, hash_kind):
    rng = np.random.default_rng(100 + 10 * dtype + hash_kind)
    n_cases = 0
    for M in (1, 2, 3):
        for N in range(1, 9):
            for _ in range(4):
                L = int(rng.integers(1, 65))
                w = _values_f32(rng, L)
                bits = synth.f32_to_bf16_bits(w).astype(np.uint32) if dtype == 1 else w.view(np.uint32).copy()
                vals = orc.value_of(bits, dtype).tolist()
                positions = rng.permutation(4 * L)[:L].astype(np.uint32)   # distinct positions
                seed, layer, t = int(rng.integers(0, 2**63)), int(rng.integers(0, 50)), int(rng.integers(0, 999))
                idx = orc.hash_indices(hash_kind, seed, layer, t, M, positions, N)
                S = brute.buckets(vals, idx, M, N)
                # oracle, with a random insertion order each time
                order = rng.permutation(L)
                cells = orc.sketch_unit(bits[order], positions[order], M, N, dtype=dtype, hash_kind=hash_kind,
                                        seed=seed, layer=layer, t=t)
                want = np.array([_to_bits([v], dtype)[0] if not math.isinf(v) else (0x7F80 if dtype else 0x7F800000)
                                 for row in S for v in row], np.uint32).reshape(M, N)
                np.testing.assert_array_equal(cells, want)
                rec = orc.retrieve_unit(cells, positions, dtype=dtype, hash_kind=hash_kind, seed=seed, layer=layer,
                                        t=t)
                want_r = _to_bits(brute.reconstruct(S, idx, M, L), dtype)
                np.testing.assert_array_equal(rec, want_r)
                n_cases += 1
    assert n_cases == 3 * 8 * 4


def test_order_independence_large(orc):
    """Any permutation of the (position, weight) multiset gives bit-identical cells."""
    rng = np.random.default_rng(7)
    L, M, N = 5000, 3, 301
    w = synth.edge_matrix_f32("mixed", 1, L, seed=5)[0]
    bits = w.view(np.uint32).copy()
    pos = np.arange(L, dtype=np.uint32)
    ref = orc.sketch_unit(bits, pos, M, N, seed=11)
    for _ in range(3):
        p = rng.permutation(L)
        np.testing.assert_array_equal(orc.sketch_unit(bits[p], pos[p], M, N, seed=11), ref)
