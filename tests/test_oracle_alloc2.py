"""Pins of the two-level (layer x row) allocation (PAPER.md:511-516 layer importance
"Front-end layers are more important"; ledger L28)."""
import numpy as np
import pytest


def test_conservation_and_proportional_share(orc):
    imp = np.array([3.0, 1.0, 2.0, 0.5])
    numel = np.array([4096, 8192, 4096, 2048])
    units = np.array([64, 64, 32, 32])
    T = 5000
    Tl = orc.layer_cells(imp, numel, units, 3, 1, T)
    assert Tl.sum() == T
    q = np.floor(imp / imp.max() * 2 ** 24)
    share = T * q * numel / np.sum(q * numel)
    assert (np.abs(Tl - share) < 1).all()  # largest remainder of the exact share


def test_uniform_importance_is_proportional_to_size(orc):
    numel = np.array([2048 * 512, 512 * 512, 8192 * 512])
    Tl = orc.layer_cells(np.ones(3), numel, np.array([512, 512, 512]), 3, 1, 100_000)
    r = Tl / numel
    assert r.max() - r.min() < 3 / numel.min()


def test_scale_invariance_and_monotonicity(orc):
    imp = np.array([0.9, 0.3, 0.6, 0.6])
    args = (np.array([1024] * 4), np.array([16] * 4), 2, 1, 3000)
    a = orc.layer_cells(imp, *args)
    b = orc.layer_cells(imp * 4.0, *args)  # exact power-of-two scaling: same fixed point
    np.testing.assert_array_equal(a, b)
    assert a[0] > a[2] == a[3] > a[1]


def test_floors_are_water_filled(orc):
    # an unimportant layer keeps exactly its floor U_l * M * min_cols; the rest is shared
    imp = np.array([1.0, 0.0, 1.0])
    Tl = orc.layer_cells(imp, np.array([1000, 1000, 1000]), np.array([10, 10, 10]), 3, 2, 600)
    assert Tl[1] == 10 * 3 * 2 and Tl.sum() == 600 and Tl[0] == Tl[2] == 270
    with pytest.raises(orc.OracleError):
        orc.layer_cells(imp, np.array([1000] * 3), np.array([10] * 3), 3, 8, 600)  # floors exceed T


def test_two_level_plan_front_layers_get_more(orc):
    # Appendix A: importance decreasing with depth -> front layers get more bits per weight; the
    # model budget holds and every layer's row allocation uses its share
    shapes = [(256, 128)] * 4
    imp = np.array([4.0, 2.0, 1.0, 0.5])
    bpw = 1.0
    pl = orc.plan(shapes, bpw, M=3, dtype=orc.BF16, seed=3, layer_importance=imp)
    budget_model = int(np.floor(bpw * 4 * 256 * 128))
    cells = [int(pl.offsets[pl.layer_units(l)[1]] - pl.offsets[pl.layer_units(l)[0]]) for l in range(4)]
    assert sum(cells) * 16 <= budget_model
    assert cells[0] > cells[1] > cells[2] > cells[3]
    for l in range(4):
        budget, meta, T, achieved = (int(x) for x in pl.acct[l])
        assert budget == T * 16 + meta and cells[l] <= T and achieved == cells[l] * 16 + meta
    T_all = orc.layer_cells(imp, np.array([256 * 128] * 4), np.array([128] * 4), 3, 1, budget_model // 16)
    np.testing.assert_array_equal(pl.acct[:, 2], T_all)
    with pytest.raises(orc.OracleError):
        orc.plan(shapes, bpw, M=3, layer_importance=imp, gran=orc.GRAN_LAYER)


def test_two_level_hand_worked_example(orc):
    # Worked by hand from ledger L28 (no code):  two [8, 4] fp32 layers, M = 1, C = 1 (no class map),
    # layer importance [1, 3], 16 bpw -> model budget 16 * 64 = 1024 bits -> T = 32 cells.
    #   q = floor((imp / 3) * 2^24) = [5592405, 16777216];  W = 32 * (5592405 + 16777216) = 32 * 22369621
    #   x_0 = 32 * 5592405 / 22369621 = 7.99999946...,  x_1 = 32 * 16777216 / 22369621 = 24.0000005...
    #   floors [7, 24] (above the U_l M min_cols = 4 floors), 1 cell left -> the larger fraction
    #   (layer 0, 0.99999946 vs 0.0000005) -> T_l = [8, 24];  rows inside a layer: 4 units of one
    #   class -> N = 2 and N = 6 columns per unit; achieved 8 * 32 + 24 * 32 = 1024 bits.
    Tl = orc.layer_cells(np.array([1.0, 3.0]), np.array([32, 32]), np.array([4, 4]), 1, 1, 32)
    np.testing.assert_array_equal(Tl, [8, 24])
    pl = orc.plan([(8, 4), (8, 4)], 16.0, M=1, dtype=orc.F32, seed=1, layer_importance=np.array([1.0, 3.0]))
    np.testing.assert_array_equal(pl.acct[:, 2], [8, 24])
    np.testing.assert_array_equal(pl.ncols, [2, 2, 2, 2, 6, 6, 6, 6])
    assert int(pl.acct[:, 3].sum()) == 1024
