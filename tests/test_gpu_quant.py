"""GPU parity of stacked state quantisation (DESIGN.md ledger L25): plans, packed
codes, fp32 group scales and reconstructions bit-exact against the CPU oracle; sketch-GEMV within
the 1e-5 scaled-error bar; bf16 prefill within 2e-2 of the fp64 oracle."""
import numpy as np
import pytest

import synth
from test_gpu_parity import DT, assert_plan_equal, make_weights, to_dev, w_bits

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def usk():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2506_17255_b200 import usk as u
    return u


def run_q(orc, usk, shapes, q, G, dtype="bf16", bpw=1.0, M=3, gran="row", g=1, C=None, saliency=None,
          hash_kind="x", seed=99, wseed=5, layer_ids=None):
    Ws = make_weights(shapes, dtype, wseed)
    sal_dev = None if saliency is None else [torch.from_numpy(s).cuda() for s in saliency]
    pl = usk.plan_allocation(shapes, bpw=bpw, rows=M, granularity=gran, dims_per_unit=g,
                             n_classes=0 if C is None else C, hash=hash_kind, dtype=dtype, seed=seed,
                             saliency=sal_dev, state_bits=q, group_size=G)
    opl = orc.plan(shapes, bpw, M=M, dtype=DT[dtype], saliency=saliency, gran=1 if gran == "layer" else 0, g=g,
                   C=C, hash_kind=0 if hash_kind == "x" else 1, seed=seed, state_bits=q, group=G)
    sk = pl.new_sketch()
    sk.fill_(0xCD)
    dW = [to_dev(W, dtype) for W in Ws]
    if layer_ids is None:
        usk.build(pl, dW, sk)
    else:  # layer-sharded: one call per id subset
        for ids in layer_ids:
            usk.build(pl, [dW[l] for l in ids], sk, layer_ids=ids)
    usk.check(pl)
    osk = orc.build_model(opl, Ws)
    return pl, opl, sk, osk, Ws


def codes_scales(sk, pl):
    a = sk.cpu().numpy()
    info = pl.info
    nb = info["total_cells"] * info["state_bits"] // 8
    off = info["scales_offset"]
    return a[:nb], a[off:off + 4 * info["n_groups"]].view(np.float32)


CASES = [
    # (shapes, q, G, dtype, bpw, M, gran, g, hash)
    ([(256, 128), (96, 64)], 4, 128, "bf16", 1.0, 3, "row", 1, "x"),
    ([(256, 128), (96, 64)], 8, 64, "bf16", 2.0, 3, "row", 1, "x"),
    ([(300, 96), (33, 64)], 4, 32, "f32", 2.0, 2, "row", 1, "x"),     # ragged tiles and rows, fp32
    ([(130, 64)], 8, 128, "bf16", 2.0, 3, "row", 2, "x"),               # dims_per_unit = 2 (generic)
    ([(96, 64), (64, 32)], 4, 64, "bf16", 2.0, 3, "layer", 1, "x"),     # LAYER granularity (generic)
    ([(70, 64)], 4, 32, "bf16", 8.0, 1, "row", 1, "identity"),
    ([(64, 256)], 4, 128, "bf16", 4.0, 5, "row", 1, "x"),               # runtime-M kernel
]


@pytest.mark.parametrize("case", CASES, ids=[f"q{c[1]}-G{c[2]}-{c[3]}-{c[6]}-g{c[7]}-M{c[5]}-{c[8]}" for c in CASES])
def test_quantised_build_reconstruct_bit_exact(orc, usk, case):
    shapes, q, G, dtype, bpw, M, gran, g, hk = case
    pl, opl, sk, osk, Ws = run_q(orc, usk, shapes, q, G, dtype, bpw, M, gran, g, hash_kind=hk)
    assert_plan_equal(pl, opl)
    assert pl.info["state_bits"] == q and pl.info["group_size"] == G
    assert pl.info["n_groups"] * G == opl.total_cells
    codes, scales = codes_scales(sk, pl)
    np.testing.assert_array_equal(codes, osk.packed)
    np.testing.assert_array_equal(scales.view(np.uint32), osk.scales.view(np.uint32))
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    for l, (o, i) in enumerate(shapes):
        Wr = torch.empty((o, i), dtype=tdt, device="cuda")
        usk.reconstruct(pl, sk, l, Wr)
        np.testing.assert_array_equal(w_bits(Wr, dtype), orc.reconstruct_rows(opl, osk, l))
        # a row sub-range through an unaligned leading dimension
        r0, r1 = o // 3, o // 3 + 5
        buf = torch.zeros((r1 - r0, i + 8), dtype=tdt, device="cuda")
        usk.reconstruct(pl, sk, l, buf[:, :i], r0, r1)
        np.testing.assert_array_equal(w_bits(buf[:, :i].contiguous(), dtype), orc.reconstruct_rows(opl, osk, l, r0, r1))


@pytest.mark.parametrize("case", CASES[:3] + CASES[5:], ids=lambda c: f"q{c[1]}-{c[3]}-M{c[5]}")
def test_quantised_gemv(orc, usk, case):
    shapes, q, G, dtype, bpw, M, gran, g, hk = case
    pl, opl, sk, osk, Ws = run_q(orc, usk, shapes, q, G, dtype, bpw, M, gran, g, hash_kind=hk)
    for l, (o, i) in enumerate(shapes):
        xv = synth.vector(i, seed=30 + l)[0]
        x = torch.from_numpy(xv.astype(np.float32)).cuda()
        y = torch.empty(o, dtype=torch.float32, device="cuda")
        usk.linear(pl, sk, l, x.view(1, -1), y.view(1, -1), usk.new_workspace(pl, l))
        y64 = orc.linear_rows(opl, osk, l, xv.astype(np.float64))[0]
        # scale of the sum: sum_j |x_j w'_oj| with w' the fp32 dequantised values
        denom = np.abs(_deq_matrix(orc, opl, osk, l)) @ np.abs(xv.astype(np.float64))
        err = np.abs(y.cpu().numpy().astype(np.float64) - y64) / np.maximum(denom, 1e-30)
        assert err.max() <= 1e-5, err.max()


def _deq_matrix(orc, opl, osk, l):
    """W' as the fp32 dequantised values (before any rounding to the weight dtype)."""
    o, i = opl.shapes[l]
    return np.stack([orc.linear_rows(opl, osk, l, np.eye(i)[j:j + 1])[0] for j in range(i)], axis=1)


def test_quantised_layer_sharded_build(orc, usk):
    shapes = [(96, 64), (128, 64), (64, 128), (40, 64)]
    pl, opl, sk, osk, Ws = run_q(orc, usk, shapes, 4, 64, "bf16", 2.0, 3, layer_ids=[[0, 2], [3, 1]])
    codes, scales = codes_scales(sk, pl)
    np.testing.assert_array_equal(codes, osk.packed)
    np.testing.assert_array_equal(scales.view(np.uint32), osk.scales.view(np.uint32))


def test_quantised_prefill(orc, usk):
    shapes = [(256, 128)]
    pl, opl, sk, osk, Ws = run_q(orc, usk, shapes, 4, 128, "bf16", 1.0, 3)
    T = 96
    X = synth.vector(128, seed=3, T=T)
    Xb = synth.f32_to_bf16_bits(X.astype(np.float32))
    x = torch.from_numpy(Xb.view(np.int16).copy()).view(torch.bfloat16).cuda()
    y = torch.empty((T, 256), dtype=torch.bfloat16, device="cuda")
    usk.linear(pl, sk, 0, x, y, usk.new_workspace(pl, 0, T))
    # reference: fp64 X (bf16 values) @ W'^T with W' the bf16-rounded reconstruction (what the
    # tensor-core path multiplies), output rounded to bf16
    Wr = orc.value_of(orc.reconstruct_rows(opl, osk, 0), orc.BF16)
    ref = synth.bf16_bits_to_f32(Xb).astype(np.float64) @ Wr.T
    got = y.float().cpu().numpy().astype(np.float64)
    rel = np.abs(got - ref).max() / np.abs(ref).max()
    assert rel <= 2e-2, rel


def test_quantised_paper_point_full_layer_sampled(orc, usk):
    # the paper's 0.5-bpw point (rate 1/8 x q4) on the Llama-3.2-1B gate shape: full-size GPU build,
    # codes/scales of the first 64 units and sampled reconstructions against the oracle
    o, i = 8192, 2048
    W = synth.weights_bf16(o, i, synth.seed_for(2, 0, 4))
    pl = usk.plan_allocation([(o, i)], bpw=0.5, rows=3, dtype="bf16", seed=0x5EED, state_bits=4, group_size=128)
    opl = orc.plan([(o, i)], 0.5, M=3, dtype=orc.BF16, seed=0x5EED, state_bits=4, group=128)
    assert_plan_equal(pl, opl)
    sk = pl.new_sketch()
    usk.build(pl, [to_dev(W, "bf16")], sk)
    usk.check(pl)
    raw = np.full(opl.total_cells, orc.inf_bits(orc.BF16), dtype=np.uint16)
    orc.build_layer(opl, 0, W, raw, 0, 64)
    cend = int(opl.offsets[64])
    gend = cend // 128  # complete groups covered by units 0..63
    codes, scales = orc.quantize(orc.BF16, raw[:gend * 128], 4, 128)
    gcodes, gscales = codes_scales(sk, pl)
    np.testing.assert_array_equal(gcodes[:gend * 64], orc.pack_codes(4, codes))
    np.testing.assert_array_equal(gscales[:gend].view(np.uint32), scales.view(np.uint32))
    # sampled reconstruction of units fully inside the verified groups
    rng = np.random.default_rng(1)
    tmax = int(np.searchsorted(opl.offsets, gend * 128, side="right")) - 2
    oj = np.stack([rng.integers(0, o, 400), rng.integers(0, max(tmax, 1), 400)], axis=1).astype(np.int64)
    qs = orc.QSketch(codes, scales, orc.pack_codes(4, codes), orc.dequantize(codes, scales, 128), raw)
    deq_full = np.zeros(opl.total_cells, dtype=np.uint32)
    deq_full[:gend * 128] = qs.deq
    qs.deq = deq_full
    want = orc.reconstruct_entries(opl, qs, 0, oj)
    Wr = torch.empty((o, i), dtype=torch.bfloat16, device="cuda")
    usk.reconstruct(pl, sk, 0, Wr)
    got = w_bits(Wr, "bf16")[oj[:, 0], oj[:, 1]]
    np.testing.assert_array_equal(got, want)


def test_two_level_allocation_plan_parity(orc, usk):
    # SURVEY 8(f4) two-level (layer x row) allocation: the device plan equals the oracle's, with
    # saliency-driven classes inside each layer (ledger L28)
    shapes = [(256, 128), (128, 256), (512, 128), (64, 64)]
    imp = [4.0, 1.5, 2.0, 0.25]
    rng = np.random.default_rng(4)
    sal = [rng.gamma(1.0, 1.0, i).astype(np.float32) for o, i in shapes]
    pl = usk.plan_allocation(shapes, bpw=1.0, rows=3, dtype="bf16", seed=6, layer_importance=imp,
                             saliency=[torch.from_numpy(s).cuda() for s in sal])
    opl = orc.plan(shapes, 1.0, M=3, dtype=orc.BF16, seed=6, layer_importance=np.array(imp), saliency=sal)
    assert_plan_equal(pl, opl)
    W = make_weights(shapes, "bf16", 2)
    sk = pl.new_sketch()
    usk.build(pl, [to_dev(w, "bf16") for w in W], sk)
    osk = orc.build_model(opl, W)
    np.testing.assert_array_equal(sk.cpu().numpy().view(np.uint16)[:opl.total_cells], osk)
