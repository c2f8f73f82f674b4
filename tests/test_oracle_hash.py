"""The hash contract USK-X.  The paper fixes only "independent hash
functions" of a storage-free address, so individual index values are our
definition ("parity unpinned"); the statistics are pinned in test_oracle_stats.py.  Here a
second implementation written from DESIGN.md's text checks the C oracle, and the frozen vectors
in tests/golden/hash_vectors.json (written by tests/golden/gen_golden.py, which calls only
oracle/) guard the contract against accidental change."""
import json
import os

import numpy as np

M64 = (1 << 64) - 1
M32 = (1 << 32) - 1


def splitmix64(x):
    x = (x + 0x9E3779B97F4A7C15) & M64
    z = x
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def fmix32(h):
    h ^= h >> 16
    h = (h * 0x85EBCA6B) & M32
    h ^= h >> 13
    h = (h * 0xC2B2AE35) & M32
    return h ^ (h >> 16)


def usk_x(seed, layer, t, row, p, N):
    rho = splitmix64((seed + 0x200 + row) & M64) & M32
    kap = splitmix64((seed + 0x300 + row) & M64) & M32
    K = splitmix64(seed ^ splitmix64((layer << 32) | t)) & M32
    h = fmix32(p ^ rho) ^ fmix32(K ^ kap)
    if N <= 1 << 16:
        return ((h % (1 << 23)) * N) // (1 << 23)
    return (h * N) // (1 << 32)


def test_contract_second_implementation(orc):
    rng = np.random.default_rng(0)
    for _ in range(3000):
        seed = int(rng.integers(0, 2**63)) * 2 + int(rng.integers(0, 2))
        layer, t = int(rng.integers(0, 300)), int(rng.integers(0, 20000))
        row, p = int(rng.integers(0, 8)), int(rng.integers(0, 2**32))
        N = int(rng.integers(1, 2**31)) if rng.integers(0, 2) else int(rng.integers(1, 2**16 + 2))
        assert orc.hash_index(0, seed, layer, t, row, p, N) == usk_x(seed, layer, t, row, p, N)
        assert orc.hash_index(1, seed, layer, t, row, p, N) == p % N


def test_frozen_vectors(orc):
    path = os.path.join(os.path.dirname(__file__), "golden", "hash_vectors.json")
    vec = json.load(open(path))
    for (seed, layer, t, row, p, N, idx) in vec["vectors"]:
        assert orc.hash_index(0, seed, layer, t, row, p, N) == idx


def test_rows_independent_of_M(orc):
    """Adding rows never changes earlier rows (needed by SPEC.md:104 row monotonicity)."""
    w = np.random.default_rng(1).standard_normal(500).astype(np.float32)
    pos = np.arange(500, dtype=np.uint32)
    c2 = orc.sketch_unit(w.view(np.uint32), pos, 2, 37, seed=4)
    c5 = orc.sketch_unit(w.view(np.uint32), pos, 5, 37, seed=4)
    np.testing.assert_array_equal(c5[:2], c2)


def test_short_unit_float_form(orc):
    """The fast GPU kernels evaluate the short-unit range reduction as one fp32 fused multiply-add
    rounded toward zero: with f = 1 + k/2^23,
    RZ(f * 4N + (2^25 - 4N + 4 off)) = 2^25 + 4 (off + floor(k N / 2^23)) whenever off + N < 2^23
    (exact product, one rounding; the result lies in [2^25, 2^26) where the fp32 ulp is 4), so the
    bit pattern is 0x4C000000 + off + idx.  Check that identity against the integer contract with the
    rounding done exactly in Python fractions."""
    from fractions import Fraction
    rng = np.random.default_rng(5)
    for _ in range(3000):
        k = int(rng.integers(0, 1 << 23))
        N = int(rng.integers(1, 1 << 16))
        off = int(rng.integers(0, (1 << 23) - N))
        exact = Fraction((1 << 23) + k, 1 << 23) * (4 * N) + ((1 << 25) - 4 * N + 4 * off)
        rz = (exact.numerator // exact.denominator) // 4 * 4  # toward zero to a multiple of the ulp 4
        assert (1 << 25) <= rz < (1 << 26)
        bits = (152 << 23) + (rz - (1 << 25)) // 4
        assert bits - 0x4C000000 - off == (k * N) >> 23
        assert (bits * 128) % (1 << 32) == ((off + ((k * N) >> 23)) * 128) % (1 << 32)


def usk_xg(seed, layer, t, row, p, N):
    """USK-XG (DESIGN.md ledger L32), from the text: USK-X with the unit key of the key group
    floor(t / 8) in place of t."""
    return usk_x(seed, layer, t // 8, row, p, N)


def test_xg_second_implementation(orc):
    rng = np.random.default_rng(11)
    for _ in range(3000):
        seed = int(rng.integers(0, 2**63))
        layer, t = int(rng.integers(0, 300)), int(rng.integers(0, 20000))
        row, p = int(rng.integers(0, 8)), int(rng.integers(0, 2**32))
        N = int(rng.integers(1, 2**31)) if rng.integers(0, 2) else int(rng.integers(1, 2**16 + 2))
        assert orc.hash_index(orc.HASH_XG, seed, layer, t, row, p, N) == usk_xg(seed, layer, t, row, p, N)


def test_xg_groups(orc):
    """The 8 units of a key group hash every position identically (for equal N); units of
    different groups, and the same unit under USK-X, hash differently (row-wise independent
    functions)."""
    pos = np.arange(4096, dtype=np.uint32)
    N = 85
    base = orc.hash_indices(orc.HASH_XG, 5, 3, 16, 3, pos, N)
    for t in range(17, 24):
        np.testing.assert_array_equal(orc.hash_indices(orc.HASH_XG, 5, 3, t, 3, pos, N), base)
    for t in (15, 24, 1000):
        assert (orc.hash_indices(orc.HASH_XG, 5, 3, t, 3, pos, N) != base).mean() > 0.9
    # group g of USK-XG is unit g of USK-X
    np.testing.assert_array_equal(base, orc.hash_indices(orc.HASH_X, 5, 3, 2, 3, pos, N))


def test_packed_float_form():
    """The packed decode kernel (L32) evaluates the short-unit reduction with the result
    at ulp 512: with f = 1 + k/2^23 and c = 2^32 + B - 512 N (B a multiple of 512, B + 512 N < 2^32),
    RZ(f * 512N + c) = 2^32 + B + 512 floor(k N / 2^23), so bits * 512 mod 2^32 = B + 512 idx -- the
    byte address of column idx in a 512-B-per-column slot row.  Checked with exact rationals."""
    from fractions import Fraction
    rng = np.random.default_rng(6)
    for _ in range(3000):
        k = int(rng.integers(0, 1 << 23))
        N = int(rng.integers(1, 1 << 16))
        B = int(rng.integers(0, ((1 << 32) - 512 * N) // 512)) * 512
        c = (1 << 32) + B - 512 * N
        # c must be an fp32 number: a multiple of its ulp (256 below 2^32, 512 above)
        assert c % (256 if c < (1 << 32) else 512) == 0 and (1 << 31) <= c < (1 << 33)
        exact = Fraction((1 << 23) + k, 1 << 23) * (512 * N) + c
        rz = (exact.numerator // exact.denominator) // 512 * 512  # toward zero, ulp 512 in [2^32, 2^33)
        assert (1 << 32) <= rz < (1 << 33)
        bits = (159 << 23) + (rz - (1 << 32)) // 512
        assert (bits * 512) % (1 << 32) == B + 512 * ((k * N) >> 23)
