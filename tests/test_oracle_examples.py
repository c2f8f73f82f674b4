"""Oracle vs the worked examples the paper / SPEC fix (tests/golden/paper_values.json)."""
import json
import os

import numpy as np
import pytest

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))
SPEC = GOLD["spec_examples"]


def f32bits(v):
    return int(np.array([v], np.float32).view(np.uint32)[0])


def f32val(b):
    return float(np.array([b], np.uint32).view(np.float32)[0])


def test_hash_identity_examples(orc):
    e = SPEC["hash_identity"]
    assert orc.hash_index(orc.HASH_IDENTITY, 0, 0, 0, 0, e["addr"], e["columns"]) == e["index"]
    e = SPEC["hash_single_column"]
    for row in range(8):
        assert orc.hash_index(orc.HASH_X, e["seed"], 0, 0, row, e["addr"], e["columns"]) == e["index"]
        assert orc.hash_index(orc.HASH_X, e["seed"], 3, 17, row, 123456, 1) == 0


def test_update_examples(orc):
    for cell, x, want in SPEC["update"]["cases"]:
        assert f32val(orc.update(orc.F32, f32bits(cell), f32bits(x))) == pytest.approx(want)
    # initialisation: +inf is replaced by any finite weight
    assert f32val(orc.update(orc.F32, 0x7F800000, f32bits(-3.5))) == -3.5
    # tie rule (L2): +x beats -x in both directions of arrival
    assert orc.update(orc.F32, f32bits(-0.25), f32bits(0.25)) == f32bits(0.25)
    assert orc.update(orc.F32, f32bits(0.25), f32bits(-0.25)) == f32bits(0.25)
    assert orc.update(orc.F32, f32bits(-0.0), f32bits(0.0)) == f32bits(0.0)


def test_retrieve_example(orc):
    e = SPEC["retrieve"]
    got = orc.retrieve(orc.F32, [f32bits(v) for v in e["bonded"]])
    assert f32val(got) == e["result"]
    # max-|.| returns the signed value (L1); tie -> non-negative (L2)
    assert f32val(orc.retrieve(orc.F32, [f32bits(0.1), f32bits(-0.7)])) == pytest.approx(-0.7)
    assert orc.retrieve(orc.F32, [f32bits(-0.5), f32bits(0.5)]) == f32bits(0.5)


def test_hand_trace(orc):
    e = SPEC["hand_trace"]
    w = np.array(e["weights"], np.float32)
    cells = orc.sketch_unit(orc.bits_of(w, orc.F32), np.arange(len(w)), e["rows"], e["columns"],
                            hash_kind=orc.HASH_IDENTITY)
    np.testing.assert_array_equal(orc.value_of(cells[0], orc.F32), np.array(e["buckets"], np.float32))
    r = orc.retrieve_unit(cells, np.arange(len(w)), hash_kind=orc.HASH_IDENTITY)
    np.testing.assert_array_equal(orc.value_of(r, orc.F32), np.array(e["retrievals"], np.float32))


@pytest.mark.parametrize("dtype", [0, 1])
def test_injective_identity(orc, dtype):
    """SPEC.md:79/98/106: identity hash, N >= L, M = 1 reproduces every weight bit-exactly."""
    rng = np.random.default_rng(3)
    L = 97
    w = rng.standard_normal(L).astype(np.float32)
    if dtype == orc.BF16:
        import synth
        bits = synth.f32_to_bf16_bits(w).astype(np.uint32)
    else:
        bits = orc.bits_of(w, orc.F32)
    for N in (L, L + 5):
        cells = orc.sketch_unit(bits, np.arange(L), 1, N, dtype=dtype, hash_kind=orc.HASH_IDENTITY)
        np.testing.assert_array_equal(orc.retrieve_unit(cells, np.arange(L), dtype=dtype,
                                                        hash_kind=orc.HASH_IDENTITY), bits)


def test_single_weight_exact(orc):
    """a single weight, any config, retrieves exactly."""
    for M in (1, 3, 8):
        for N in (1, 7):
            cells = orc.sketch_unit([f32bits(-1.25)], [11], M, N, seed=99)
            assert orc.retrieve_unit(cells, [11], seed=99)[0] == f32bits(-1.25)
            # every other cell keeps the +inf sentinel
            assert (cells == 0x7F800000).sum() == M * N - M


def test_nonfinite_rejected(orc):
    with pytest.raises(orc.OracleError) as ei:
        orc.sketch_unit([f32bits(1.0), 0x7FC00000], [0, 1], 2, 4)
    assert ei.value.status == orc.ENONFINITE


def test_importance_example(orc):
    e = SPEC["importance"]
    np.testing.assert_allclose(orc.importance(np.array(e["samples"], np.float32)), e["I"], rtol=0, atol=0)
    # constant activation c -> c^2
    np.testing.assert_allclose(orc.importance(np.full((7, 3), 1.5, np.float32)), [2.25] * 3)


def test_allocation_examples(orc):
    cases = SPEC["allocation"]["cases"]
    for c in cases[:2]:
        ncols, _ = orc.allocate(c["scores"], c["budget"], min_cols=c["floor"])
        assert ncols.tolist() == c["cols"]
    c = cases[2]
    ncols, _ = orc.allocate(c["scores"], c["budget"], min_cols=c["floor"])
    assert ncols[0] == c["zero_unit_cols"]
    assert ncols.sum() <= c["budget"]
    with pytest.raises(orc.OracleError) as ei:  # infeasible floor
        orc.allocate([1, 1, 1], 40, min_cols=16)
    assert ei.value.status == orc.EBUDGET


def test_peak_memory_example(orc):
    e = SPEC["peak_memory"]
    assert orc.peak_memory(e["layers"], e["sketches"]) == e["estimate"]
    assert sum(e["layers"]) == e["baseline"]


def test_table1_bit_arithmetic(orc):
    """Equivalent bits = rate x state bits.  Our plans store raw states,
    so a plan at `bpw` with 16-bit states has rate bpw/16 and its achieved bits stay <= budget."""
    for rate, qbits, eq in GOLD["table1_equivalent_bits"]["rows"]:
        assert rate * qbits == eq
    # 0.5 bpw with raw bf16 states is rate 1/32; the achieved bits/weight never exceed the budget
    pl = orc.plan([(256, 512)], 0.5, M=3, dtype=orc.BF16)
    budget, meta, T, achieved = pl.acct[0]
    assert budget == int(np.floor(0.5 * 256 * 512))
    assert achieved == pl.total_cells * 16 + meta
    assert achieved <= budget
    pl = orc.plan([(256, 512)], 8.0, M=1, dtype=orc.BF16)  # rate 1/2 of 16-bit states
    assert pl.total_cells == 256 * 512 // 2
