"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, on the same seeded inputs.

Bar: plan arrays, sketch bytes and reconstructions bit-exact; sketch-GEMV
within max_o |y - y64| / sum_j |x_j w'_oj| <= 1e-5 (fp32 accumulation vs the oracle's fp64)."""
import numpy as np
import pytest

import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def usk():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2506_17255_b200 import usk as u
    return u


DT = {"bf16": 1, "f32": 0}


def to_dev(W, dtype):
    if dtype == "bf16":
        return torch.from_numpy(W.view(np.int16).copy()).view(torch.bfloat16).cuda()
    return torch.from_numpy(np.ascontiguousarray(W, np.float32)).cuda()


def sketch_cells(sk, pl_dev, dtype):
    a = sk.cpu().numpy()
    n = pl_dev.info["total_cells"]
    return a.view(np.uint16)[:n] if dtype == "bf16" else a.view(np.uint32)[:n]


def w_bits(t, dtype):
    a = t.cpu()
    return a.view(torch.int16).numpy().view(np.uint16) if dtype == "bf16" else a.numpy().view(np.uint32)


def make_weights(shapes, dtype, seed, kind=None):
    out = []
    for k, (o, i) in enumerate(shapes):
        if kind is not None:
            W = synth.edge_matrix_bf16(kind, o, i, seed + k) if dtype == "bf16" else synth.edge_matrix_f32(kind, o, i, seed + k)
        elif dtype == "bf16":
            W = synth.weights_bf16(o, i, seed + k)
        else:
            W = synth.weights_f32(o, i, seed + k)
        out.append(W)
    return out


def run_both(orc, usk, shapes, dtype="bf16", bpw=0.5, M=3, gran="row", g=1, C=None, saliency=None,
             hash_kind="x", seed=1234, kind=None, wseed=7):
    Ws = make_weights(shapes, dtype, wseed, kind)
    sal_dev = None if saliency is None else [torch.from_numpy(s).cuda() for s in saliency]
    pl = usk.plan_allocation(shapes, bpw=bpw, rows=M, granularity=gran, dims_per_unit=g,
                             n_classes=0 if C is None else C, hash=hash_kind, dtype=dtype, seed=seed,
                             saliency=sal_dev)
    opl = orc.plan(shapes, bpw, M=M, dtype=DT[dtype], saliency=saliency, gran=1 if gran == "layer" else 0, g=g,
                   C=C, hash_kind=0 if hash_kind == "x" else 1, seed=seed)
    sk = pl.new_sketch()
    sk.fill_(0xAB)
    dW = [to_dev(W, dtype) for W in Ws]
    usk.build(pl, dW, sk)
    usk.check(pl)
    osk = orc.build_model(opl, Ws)
    return pl, opl, sk, osk, Ws, dW


def assert_plan_equal(pl, opl):
    for l in range(len(opl.shapes)):
        cls, ncols, nrows, offs = pl.export(l)
        u0, u1 = opl.layer_units(l)
        np.testing.assert_array_equal(cls, opl.cls[u0:u1])
        np.testing.assert_array_equal(ncols, opl.ncols[u0:u1])
        np.testing.assert_array_equal(offs, opl.offsets[u0:u1 + 1])
        np.testing.assert_array_equal(nrows, opl.nrows[u0:u1])
        li = pl.layers[l]
        assert li.budget_bits == opl.acct[l, 0] and li.meta_bits == opl.acct[l, 1]
        if opl.gran == 0:
            assert li.cells_T == opl.acct[l, 2] and li.achieved_bits == opl.acct[l, 3]
    assert pl.info["total_cells"] == opl.total_cells


CASES = [
    # (shapes, dtype, bpw, M, gran, g, hash)
    ([(256, 256)], "f32", 1.0, 2, "layer", 1, "x"),          # config 1, LAYER
    ([(256, 256)], "f32", 1.0, 2, "row", 1, "x"),            # config 1, ROW
    ([(100, 200), (64, 128)], "bf16", 1.0, 3, "row", 1, "x"),  # ragged unit tile (200 % 64 = 8), ragged rows
    ([(300, 96), (33, 64)], "bf16", 2.0, 1, "row", 1, "x"),
    ([(77, 96)], "f32", 4.0, 4, "row", 1, "x"),               # runtime-M kernel
    ([(130, 64)], "bf16", 1.0, 3, "row", 2, "x"),             # dims_per_unit = 2 (generic path)
    ([(96, 64), (64, 32)], "bf16", 1.0, 3, "layer", 1, "x"),  # LAYER bf16 (16-bit CAS path)
    ([(70, 64)], "bf16", 8.0, 1, "row", 1, "identity"),       # SPEC test hash
    ([(64, 256)], "bf16", 4.0, 5, "row", 1, "x"),
]


@pytest.mark.parametrize("case", CASES, ids=[f"{c[1]}-{c[4]}-g{c[5]}-M{c[3]}-{c[6]}-{c[0][0]}" for c in CASES])
def test_build_and_reconstruct_bit_exact(orc, usk, case):
    shapes, dtype, bpw, M, gran, g, hk = case
    pl, opl, sk, osk, Ws, dW = run_both(orc, usk, shapes, dtype, bpw, M, gran, g, hash_kind=hk)
    assert_plan_equal(pl, opl)
    np.testing.assert_array_equal(sketch_cells(sk, pl, dtype), osk)
    for l, (o, i) in enumerate(shapes):
        tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
        Wr = torch.empty((o, i), dtype=tdt, device="cuda")
        usk.reconstruct(pl, sk, l, Wr)
        np.testing.assert_array_equal(w_bits(Wr, dtype), orc.reconstruct_rows(opl, osk, l))
        # row sub-range into a strided buffer
        r0, r1 = o // 3, o - 1
        buf = torch.zeros((r1 - r0, i + 8), dtype=tdt, device="cuda")
        usk.reconstruct(pl, sk, l, buf, r0, r1)
        np.testing.assert_array_equal(w_bits(buf[:, :i].contiguous(), dtype), orc.reconstruct_rows(opl, osk, l, r0, r1))


@pytest.mark.parametrize("kind", ["pm_pairs", "zeros", "subnormal", "all_equal", "mixed", "outlier"])
@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_edge_values_bit_exact(orc, usk, kind, dtype):
    shapes = [(96, 128)]
    for gran in ("row", "layer"):
        pl, opl, sk, osk, Ws, dW = run_both(orc, usk, shapes, dtype, 2.0, 3, gran, kind=kind)
        np.testing.assert_array_equal(sketch_cells(sk, pl, dtype), osk)
        tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
        Wr = torch.empty(shapes[0], dtype=tdt, device="cuda")
        usk.reconstruct(pl, sk, 0, Wr)
        np.testing.assert_array_equal(w_bits(Wr, dtype), orc.reconstruct_rows(opl, osk, 0))


def test_plan_with_saliency_classes(orc, usk):
    shapes = synth.mlp_block_1b_shapes()
    sal = [synth.saliency_like(i, 100 + k) for k, (o, i) in enumerate(shapes)]
    pl, opl, sk, osk, Ws, dW = run_both(orc, usk, shapes, "bf16", 0.5, 3, saliency=sal, C=4, wseed=11)
    assert_plan_equal(pl, opl)
    assert len(set(opl.ncols.tolist())) > 1
    np.testing.assert_array_equal(sketch_cells(sk, pl, "bf16"), osk)


def test_plan_variants_match_oracle(orc, usk):
    rng = np.random.default_rng(0)
    shapes = synth.llama_block(2048, 512, 8192)
    for C in (1, 2, 4, 7):
        sal = [np.where(rng.random(i) < 0.05, 0.0, rng.exponential(size=i)).astype(np.float32) for (o, i) in shapes]
        pl = usk.plan_allocation(shapes, bpw=0.8, rows=3, n_classes=C, saliency=[torch.from_numpy(s).cuda() for s in sal])
        assert_plan_equal(pl, orc.plan(shapes, 0.8, M=3, saliency=sal, C=C))
    shapes8 = synth.llama_block(4096, 1024, 14336)
    assert_plan_equal(usk.plan_allocation(shapes8, bpw=0.5), orc.plan(shapes8, 0.5, M=3))
    pl = usk.plan_allocation(shapes, bpw=0.5, granularity="layer", n_classes=3,
                             saliency=[torch.from_numpy(s).cuda() for s in sal])
    assert_plan_equal(pl, orc.plan(shapes, 0.5, M=3, saliency=sal, gran=1, C=3))


def gemv_err(y, y64, x, Wr):
    scale = np.abs(x)[None, :] @ np.abs(Wr).T  # sum_j |x_j w'_oj|
    scale = np.maximum(scale, 1e-30)
    return float(np.max(np.abs(y - y64) / scale))


@pytest.mark.parametrize("case", CASES, ids=[f"{c[1]}-{c[4]}-g{c[5]}-M{c[3]}-{c[6]}-{c[0][0]}" for c in CASES])
def test_gemv_tolerance_and_determinism(orc, usk, case):
    shapes, dtype, bpw, M, gran, g, hk = case
    pl, opl, sk, osk, Ws, dW = run_both(orc, usk, shapes, dtype, bpw, M, gran, g, hash_kind=hk)
    for l, (o, i) in enumerate(shapes):
        for xdt in (("bf16", "f32") if dtype == "bf16" else ("f32",)):
            x = synth.vector(i, seed=l + 3)[0]
            if xdt == "bf16":
                xb = synth.f32_to_bf16_bits(x)
                xd = torch.from_numpy(xb.view(np.int16).copy()).view(torch.bfloat16).cuda()
                x64 = synth.bf16_bits_to_f32(xb).astype(np.float64)
            else:
                xd = torch.from_numpy(x).cuda()
                x64 = x.astype(np.float64)
            ws = usk.new_workspace(pl, l)
            y = torch.empty(o, dtype=torch.float32, device="cuda")
            usk.linear(pl, sk, l, xd.view(1, -1), y.view(1, -1), ws)
            y64 = orc.linear_rows(opl, osk, l, x64)[0]
            Wr = orc.value_of(orc.reconstruct_rows(opl, osk, l), DT[dtype]).reshape(o, i)
            err = gemv_err(y.cpu().numpy().astype(np.float64), y64, x64, Wr)
            assert err <= 1e-5, err
            # deterministic and workspace left reusable
            y2 = torch.empty_like(y)
            usk.linear(pl, sk, l, xd.view(1, -1), y2.view(1, -1), ws)
            assert torch.equal(y, y2)
            # output shards equal the full result bit-for-bit (output-sharded decode):
            # every row is summed by one fixed tree whatever the range, its start or the subtile
            # height the launch picks (query.cu transpose_reduce), so any boundary works
            for h, e in ((o // 2, o), (o // 3 + 1, o - 5), (7, min(o, 7 + 40))):
                if e <= h:
                    continue
                ys = torch.empty(e - h, dtype=torch.float32, device="cuda")
                ws2 = usk.new_workspace(pl, l, 1, h, e)
                usk.linear(pl, sk, l, xd.view(1, -1), ys.view(1, -1), ws2, out_begin=h, out_end=e)
                assert torch.equal(ys, y[h:e]), (h, e)


def test_nonfinite_weight_reported(usk):
    for dtype, gran in (("bf16", "row"), ("f32", "row"), ("bf16", "layer")):
        W = synth.weights_f32(64, 64, 1)
        W[5, 7] = np.inf if gran == "row" else np.nan
        dev = to_dev(synth.f32_to_bf16_bits(W) if dtype == "bf16" else W, dtype)
        pl = usk.plan_allocation([(64, 64)], bpw=2.0, dtype=dtype, granularity=gran)
        sk = pl.new_sketch()
        usk.build(pl, [dev], sk)
        with pytest.raises(usk.UskError) as e:
            usk.check(pl)
        assert e.value.status == usk.ENONFINITE
        usk.check(pl)  # cleared


def test_error_codes(usk):
    with pytest.raises(usk.UskError) as e:
        usk.plan_allocation([(512, 2048)], bpw=0.5, rows=3, min_cols=16)
    assert e.value.status == usk.EBUDGET
    pl = usk.plan_allocation([(64, 64)], bpw=2.0)
    sk = pl.new_sketch()
    W = torch.zeros((64, 64), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(usk.UskError) as e:
        usk.build(pl, [W], sk, layer_ids=[3])
    assert e.value.status == usk.ESHAPE
    with pytest.raises(usk.UskError) as e:
        usk.reconstruct(pl, sk, 0, W, 10, 65)
    assert e.value.status == usk.ESHAPE
    x = torch.zeros((1, 64), dtype=torch.bfloat16, device="cuda")
    y = torch.zeros((1, 64), dtype=torch.float32, device="cuda")
    with pytest.raises(usk.UskError) as e:
        usk.linear(pl, sk, 0, x, y, torch.zeros(0, dtype=torch.uint8, device="cuda"))
    assert e.value.status == usk.ESHAPE
    plf = usk.plan_allocation([(64, 64)], bpw=2.0, dtype="f32")
    with pytest.raises(usk.UskError) as e:
        usk.linear(plf, plf.new_sketch(), 0, torch.zeros((4, 64), device="cuda"), torch.zeros((4, 64), device="cuda"),
                   usk.new_workspace(plf, 0, 4))
    assert e.value.status == usk.EUNSUPPORTED


def test_importance_kernel(orc, usk):
    A = synth.activations(512, 2048, seed=5)
    I = torch.empty(2048, dtype=torch.float32, device="cuda")
    usk.importance(torch.from_numpy(A).cuda(), I)
    np.testing.assert_allclose(I.cpu().numpy(), orc.importance(A), rtol=2e-7, atol=0)
    # the SPEC example
    I2 = torch.empty(2, dtype=torch.float32, device="cuda")
    usk.importance(torch.tensor([[1.0, 0.0], [0.0, 2.0]], device="cuda"), I2)
    assert I2.cpu().tolist() == [0.5, 2.0]


def test_layer_sharded_build_equals_full(orc, usk):
    """Layer-sharded build (each 'rank' builds a disjoint layer subset into its own buffer) gives
    the same bytes per layer region as the single build (multi-GPU build)."""
    shapes = synth.llama_block(256, 64, 512)
    Ws = make_weights(shapes, "bf16", 3)
    dW = [to_dev(W, "bf16") for W in Ws]
    pl = usk.plan_allocation(shapes, bpw=2.0, seed=9)
    full = pl.new_sketch()
    usk.build(pl, dW, full)
    parts = []
    P = 3
    for r in range(P):
        ids = [l for l in range(len(shapes)) if l % P == r]
        sk = pl.new_sketch()
        sk.zero_()
        usk.build(pl, [dW[l] for l in ids], sk, layer_ids=ids)
        parts.append((ids, sk))
    for ids, sk in parts:
        for l in ids:
            li = pl.layers[l]
            a = full.view(torch.int16)[li.cell_begin:li.cell_begin + li.n_cells]
            b = sk.view(torch.int16)[li.cell_begin:li.cell_begin + li.n_cells]
            assert torch.equal(a, b)


def test_linear_batch_equals_single(orc, usk):
    """usk_linear_batch (one launch for linears sharing x) == per-linear usk_linear, bit for bit,
    and within the GEMV tolerance of the oracle; with and without output ranges."""
    shapes = synth.llama_block(256, 64, 512)[:3] + [(96, 256)]
    Ws = make_weights(shapes, "bf16", 21)
    pl = usk.plan_allocation(shapes, bpw=2.0, seed=4)
    opl = orc.plan(shapes, 2.0, M=3, dtype=orc.BF16, seed=4)
    sk = pl.new_sketch()
    usk.build(pl, [to_dev(W, "bf16") for W in Ws], sk)
    osk = orc.build_model(opl, Ws)
    xb = synth.f32_to_bf16_bits(synth.vector(256, seed=9)[0])
    x = torch.from_numpy(xb.view(np.int16).copy()).view(torch.bfloat16).cuda()
    x64 = synth.bf16_bits_to_f32(xb).astype(np.float64)
    layers = [0, 1, 2, 3]
    for ranges in (None, [(10, 200), (0, 64), (5, 6), (0, 96)]):
        rg = ranges or [(0, shapes[l][0]) for l in layers]
        ys = [torch.empty(r1 - r0, dtype=torch.float32, device="cuda") for r0, r1 in rg]
        usk.linear_batch(pl, sk, layers, x, ys, usk.new_batch_workspace(pl, layers, ranges), ranges=ranges)
        for k, l in enumerate(layers):
            r0, r1 = rg[k]
            y1 = torch.empty(r1 - r0, dtype=torch.float32, device="cuda")
            usk.linear(pl, sk, l, x.view(1, -1), y1.view(1, -1), usk.new_workspace(pl, l, 1, r0, r1), r0, r1)
            y64 = orc.linear_rows(opl, osk, l, x64, r0, r1)[0]
            Wr = orc.value_of(orc.reconstruct_rows(opl, osk, l, r0, r1), orc.BF16).reshape(r1 - r0, -1)
            assert gemv_err(ys[k].cpu().numpy().astype(np.float64), y64, x64, Wr) <= 1e-5
            assert torch.equal(ys[k], y1)  # grouped == single, with or without ranges
