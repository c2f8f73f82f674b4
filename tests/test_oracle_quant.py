"""Pins of the stacked state quantisation oracle (Table 1
"+ q4"/"+ q8"; scheme and worked examples from SPEC.md's quant module)."""
import numpy as np
import pytest
import torch

import synth


def f32(x):
    return np.float32(x)


def raw_f32(vals):
    return np.asarray(vals, dtype=np.float32).view(np.uint32)


def test_spec_example_q8(orc):
    # SPEC: group {0.5, -0.25}, 8-bit -> scale = 0.5/127, codes {127, -64} (round half away)
    codes, scales = orc.quantize(orc.F32, raw_f32([0.5, -0.25]), 8, 2)
    assert scales[0] == f32(0.5) / f32(127)
    assert codes.tolist() == [127, -64]
    # round trip -> {0.5, -0.2520}
    deq = orc.dequantize(codes, scales, 2).view(np.float32)
    assert deq[0] == f32(0.5) and abs(deq[1] - (-0.2520)) < 5e-5
    assert deq[1] == f32(-64) * scales[0]


def test_unoccupied_and_zero_groups(orc):
    inf = raw_f32([np.inf] * 4)
    codes, scales = orc.quantize(orc.F32, inf, 4, 4)
    assert scales.tolist() == [0.0] and codes.tolist() == [0, 0, 0, 0]
    zeros = raw_f32([0.0, -0.0, 0.0, 0.0])
    codes, scales = orc.quantize(orc.F32, zeros, 8, 4)
    assert scales.tolist() == [0.0] and codes.tolist() == [0, 0, 0, 0]
    # mixed: the absmax runs over occupied cells only; unoccupied cells code 0
    mixed = raw_f32([np.inf, 1.0, -3.5, np.inf])
    codes, scales = orc.quantize(orc.F32, mixed, 4, 4)
    assert scales[0] == f32(3.5) / f32(7)
    assert codes.tolist() == [0, 2, -7, 0]
    deq = orc.dequantize(codes, scales, 4).view(np.float32)
    assert deq[0] == 0.0 and deq[3] == 0.0


@pytest.mark.parametrize("q", [4, 8])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_roundtrip_error_bound(orc, q, dtype):
    # SPEC invariant: |dequant - original| <= scale/2 on every occupied element (exhaustive), up
    # to the fp32 rounding of v/scale and of code*scale (<= 2 * qmax * 2^-24 * scale; L25)
    rng = np.random.default_rng(7 + q)
    G = 128
    n = 64 * G
    v = (rng.standard_normal(n) * 0.02).astype(np.float32)
    v[rng.random(n) < 0.05] = np.inf  # unoccupied cells
    if dtype == "bf16":
        raw = synth.f32_to_bf16_bits(v)
        dt = orc.BF16
        vals = synth.bf16_bits_to_f32(raw).astype(np.float64)
    else:
        raw = v.view(np.uint32)
        dt = orc.F32
        vals = v.astype(np.float64)
    codes, scales = orc.quantize(dt, raw, q, G)
    qmax = 7 if q == 4 else 127
    assert np.all(np.abs(codes.astype(np.int64)) <= qmax)
    deq = orc.dequantize(codes, scales, G).view(np.float32).astype(np.float64)
    occ = np.isfinite(vals)
    sc = np.repeat(scales.astype(np.float64), G)
    err = np.abs(deq - np.where(occ, vals, 0.0))
    assert np.all(err[occ] <= sc[occ] * (0.5 + 2 * qmax * 2.0 ** -24) + 1e-30)
    assert np.all(deq[~occ] == 0.0)
    # the group's absmax element is coded +-qmax exactly
    for g in range(0, 64, 9):
        blk = np.where(occ[g * G:(g + 1) * G], np.abs(vals[g * G:(g + 1) * G]), -1)
        k = int(np.argmax(blk))
        assert abs(int(codes[g * G + k])) == qmax


def test_pack_codes_nibble_order(orc):
    c = np.array([1, -1, 7, -8 + 1, 0, 3], dtype=np.int8)
    b = orc.pack_codes(4, c)
    assert b.tolist() == [0xF1, 0x97, 0x30]  # even cell in the low nibble (SPEC)
    assert orc.pack_codes(8, np.array([127, -64], dtype=np.int8)).tolist() == [127, 0xC0]


def test_bf16_rne_matches_torch(orc):
    rng = np.random.default_rng(3)
    v = np.concatenate([rng.standard_normal(2000).astype(np.float32) * 0.05,
                        np.array([1.0 + 2 ** -8, 1.0 + 3 * 2 ** -8, -1.0 - 2 ** -8, 0.0, -0.0, 1e-30],
                                 dtype=np.float32)])
    ours = orc.f32_to_bf16_rne(v.view(np.uint32))
    ref = torch.from_numpy(v).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(ours, ref)


@pytest.mark.parametrize("q", [4, 8])
def test_plan_accounting_and_alignment(orc, q):
    shapes = [(96, 64), (40, 96), (64, 64)]
    G = 64
    bpw = 2.5
    pl = orc.plan(shapes, bpw, M=3, dtype=orc.BF16, state_bits=q, group=G, seed=5)
    for l, (o, i) in enumerate(shapes):
        budget, meta, T, achieved = (int(x) for x in pl.acct[l])
        assert budget == int(np.floor(bpw * o * i)) and meta == 0
        assert T == ((budget - meta) // (q * G + 32)) * G
        u0, u1 = pl.layer_units(l)
        cells = int(pl.offsets[u1] - pl.offsets[u0])
        assert cells <= T
        assert achieved == -(-cells // G) * (q * G + 32) + meta <= budget
        assert int(pl.offsets[u0]) % G == 0  # groups never straddle layers
    assert pl.total_cells % G == 0
    with pytest.raises(orc.OracleError):
        orc.plan(shapes, bpw, M=3, state_bits=4, group=48)


def test_paper_point_rate(orc):
    # Table 1 "1/8 Compression + q4" = 0.5 equivalent bits: at 0.5 bpw with
    # q4 and G = 128 a layer holds (0.5 / 4.25) cells per weight = rate 1/8.5 (the fp32 scale per
    # 128 cells costs 0.25 bits per cell; ledger L25)
    o, i = 2048, 512
    pl = orc.plan([(o, i)], 0.5, M=3, dtype=orc.BF16, state_bits=4, group=128)
    budget, meta, T, achieved = (int(x) for x in pl.acct[0])
    assert T == (budget // (4 * 128 + 32)) * 128
    assert abs(T / (o * i) - 1 / 8.5) < 1e-3
    assert achieved <= budget


def test_quantised_retrieval_brute(orc):
    # tiny matrix: W' from the oracle == max-|.| over the M dequantised bonded cells (ties ->
    # non-negative), rounded RNE to bf16, recomputed here from the hash table
    o, i, M = 24, 64, 3
    shapes = [(o, i)]
    W = synth.weights_bf16(o, i, 11)
    pl = orc.plan(shapes, 3.0, M=M, dtype=orc.BF16, state_bits=4, group=32, seed=9)
    qs = orc.build_model(pl, [W])
    rec = orc.reconstruct_rows(pl, qs, 0)
    deq = qs.deq.view(np.float32)
    for t in range(i):
        N = int(pl.ncols[t])
        off = int(pl.offsets[t])
        idx = orc.hash_indices(orc.HASH_X, 9, 0, t, M, np.arange(o), N)
        for p in range(o):
            vals = [deq[off + r * N + idx[r, p]] for r in range(M)]
            best = vals[0]
            for v in vals[1:]:
                if abs(v) > abs(best) or (abs(v) == abs(best) and best < 0 <= v):
                    best = v
            want = orc.f32_to_bf16_rne(np.array([np.float32(best).view(np.uint32)]))[0]
            assert rec[p, t] == want
    # the linear uses the fp32 dequantised values
    x = synth.vector(i, seed=2)[0].astype(np.float64)
    y = orc.linear_rows(pl, qs, 0, x)[0]
    Wq = np.zeros((o, i))
    for t in range(i):
        N = int(pl.ncols[t])
        off = int(pl.offsets[t])
        idx = orc.hash_indices(orc.HASH_X, 9, 0, t, M, np.arange(o), N)
        for p in range(o):
            vals = [float(deq[off + r * N + idx[r, p]]) for r in range(M)]
            Wq[p, t] = max(vals, key=lambda v: (abs(v), v >= 0))
    assert np.allclose(y, Wq @ x, rtol=0, atol=1e-12)
