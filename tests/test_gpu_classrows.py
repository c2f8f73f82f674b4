"""GPU parity of per-class sketch rows (SURVEY §8(f4) "Per-class row counts M_c"; north star "salient
weights more rows or buckets"; categories PAPER.md:523-528; ledger L30): plan arrays (incl. the
per-unit row counts), sketch bytes and reconstructions bit-exact against the oracle; sketch-GEMV
within the 1e-5 bar; grouped calls, Top-K, aggregated gradient and the compression report on the
same plans; prefill through the tensor-core path."""
import numpy as np
import pytest

import synth
from test_gpu_parity import DT, assert_plan_equal, gemv_err, make_weights, sketch_cells, to_dev, w_bits

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def usk():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2506_17255_b200 import usk as u
    return u


CASES = [
    # (shapes, dtype, bpw, class_rows, gran, g, topk)
    ([(200, 136), (72, 264)], "bf16", 1.0, (3, 2, 1), "row", 1, 0),      # fast kernels (M = 3), ragged tiles
    ([(160, 96)], "f32", 2.0, (1, 2), "row", 1, 0),                       # fast kernels (M = 2), fp32
    ([(96, 200)], "bf16", 2.0, (5, 3, 2, 1), "row", 1, 0),                # runtime-M fast kernels (max 5)
    ([(130, 64)], "bf16", 2.0, (3, 1), "row", 2, 0),                       # dims_per_unit = 2: generic paths
    ([(64, 48), (40, 96), (96, 32)], "f32", 1.0, (3, 2, 1), "layer", 1, 0),  # LAYER units: generic paths
    ([(256, 128)], "bf16", 2.0, (3, 2, 2, 1), "row", 1, 30),               # with Top-K outliers
]
IDS = [f"{c[1]}-{c[4]}-g{c[5]}-rows{''.join(map(str, c[3]))}-K{c[6]}" for c in CASES]


def _sal(shapes, gran):
    if gran == "layer":  # layer score = mean row importance: distinct per layer
        return [np.full(i, 2.0 ** -k, np.float32) for k, (o, i) in enumerate(shapes)]
    return [synth.saliency_like(i, 300 + k) for k, (o, i) in enumerate(shapes)]


def _both(orc, usk, case, wseed=5):
    shapes, dtype, bpw, rows, gran, g, K = case
    C = len(rows)
    sal = _sal(shapes, gran)
    Ws = make_weights(shapes, dtype, wseed)
    pl = usk.plan_allocation(shapes, bpw=bpw, rows=3, granularity=gran, dims_per_unit=g, n_classes=C, dtype=dtype,
                             seed=77, saliency=[torch.from_numpy(s).cuda() for s in sal], class_rows=rows, topk=K)
    opl = orc.plan(shapes, bpw, M=3, dtype=DT[dtype], saliency=sal, gran=1 if gran == "layer" else 0, g=g, C=C,
                   seed=77, class_rows=rows, topk=K)
    sk = pl.new_sketch()
    sk.fill_(0x5A)
    dW = [to_dev(W, dtype) for W in Ws]
    usk.build(pl, dW, sk)
    usk.check(pl)
    osk = orc.build_model(opl, Ws)
    return pl, opl, sk, osk, Ws, dW


@pytest.mark.parametrize("case", CASES, ids=IDS)
def test_classrows_build_reconstruct_gemv(orc, usk, case):
    shapes, dtype, bpw, rows, gran, g, K = case
    pl, opl, sk, osk, Ws, dW = _both(orc, usk, case)
    assert_plan_equal(pl, opl)
    assert pl.info["rows"] == max(rows)
    assert len(set(opl.nrows.tolist())) > 1                      # the plan really mixes row counts
    cells = osk.cells if K else osk
    np.testing.assert_array_equal(sketch_cells(sk, pl, dtype), cells)
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    for l, (o, i) in enumerate(shapes):
        Wr = torch.empty((o, i), dtype=tdt, device="cuda")
        usk.reconstruct(pl, sk, l, Wr)
        want = orc.reconstruct_rows(opl, osk, l)
        np.testing.assert_array_equal(w_bits(Wr, dtype), want)
        wv = orc.value_of(want, DT[dtype]).reshape(o, i)
        wo = orc.value_of(w_bits(dW[l], dtype), DT[dtype]).reshape(o, i)
        if not K:
            assert (np.abs(wv) <= np.abs(wo)).all()                # underestimate on every weight
        x = synth.vector(i, seed=40 + l)[0]
        x64 = x.astype(np.float64)
        xd = torch.from_numpy(x).cuda()
        if dtype == "bf16":
            xb = synth.f32_to_bf16_bits(x)
            xd = torch.from_numpy(xb.view(np.int16).copy()).view(torch.bfloat16).cuda()
            x64 = synth.bf16_bits_to_f32(xb).astype(np.float64)
        y = torch.empty(o, dtype=torch.float32, device="cuda")
        usk.linear(pl, sk, l, xd.view(1, -1), y.view(1, -1), usk.new_workspace(pl, l))
        y64 = orc.linear_rows(opl, osk, l, x64)[0]
        assert gemv_err(y.cpu().numpy().astype(np.float64), y64, x64, wv) <= 1e-5


def test_classrows_batch_and_shards(orc, usk):
    """q|k|v-style grouped call (shared x) on a mixed-rows plan: equal to the per-layer calls."""
    shapes = [(192, 128), (64, 128), (64, 128)]
    case = (shapes, "bf16", 1.0, (4, 3, 2, 1), "row", 1, 0)
    pl, opl, sk, osk, Ws, dW = _both(orc, usk, case)
    np.testing.assert_array_equal(sketch_cells(sk, pl, "bf16"), osk)
    x = synth.torch_vector(128, 9, "cuda", torch.bfloat16)
    ys = [torch.empty(o, dtype=torch.float32, device="cuda") for o, _ in shapes]
    usk.linear_batch(pl, sk, [0, 1, 2], x.view(1, -1), [y.view(1, -1) for y in ys],
                     usk.new_batch_workspace(pl, [0, 1, 2]))
    x64 = x.float().cpu().numpy().astype(np.float64).ravel()
    for l, (o, i) in enumerate(shapes):
        y64 = orc.linear_rows(opl, osk, l, x64)[0]
        wv = orc.value_of(orc.reconstruct_rows(opl, osk, l), 1).reshape(o, i)
        assert gemv_err(ys[l].cpu().numpy().astype(np.float64), y64, x64, wv) <= 1e-5


def test_classrows_grad_and_stats(orc, usk):
    case = ([(128, 96)], "bf16", 2.0, (3, 2, 1), "row", 1, 0)
    pl, opl, sk, osk, Ws, dW = _both(orc, usk, case)
    G = synth.weights_f32(128, 96, seed=13, scale=1e-3)
    gd = torch.from_numpy(G).cuda()
    cg = torch.empty(pl.layers[0].n_cells, dtype=torch.float32, device="cuda")
    usk.aggregate_grad(pl, 0, gd, cg)
    np.testing.assert_array_equal(cg.cpu().numpy().view(np.uint32),
                                  orc.aggregate_grad(opl, 0, G.astype(np.float64)).view(np.uint32))
    got = usk.stats(pl, sk, 0, dW[0])
    want = orc.stats(opl, 0, Ws[0], orc.reconstruct_rows(opl, osk, 0))
    for k, v in want.items():
        assert got[k] == v, (k, got[k], v)


def test_classrows_mlp_block_sampled(orc, usk):
    """BASELINE config 2 shapes (Llama-3.2-1B MLP block, 0.5 bpw, importance classes) with per-class
    rows (4, 3, 3, 2): plan equal, whole sketch bit-exact, sampled reconstructions and GEMV rows."""
    shapes = synth.mlp_block_1b_shapes()
    sal = [synth.saliency_like(i, 100 + k) for k, (o, i) in enumerate(shapes)]
    rows = (4, 3, 3, 2)
    Ws = make_weights(shapes, "bf16", 11)
    pl = usk.plan_allocation(shapes, bpw=0.5, rows=3, n_classes=4, seed=3, class_rows=rows,
                             saliency=[torch.from_numpy(s).cuda() for s in sal])
    opl = orc.plan(shapes, 0.5, M=3, saliency=sal, C=4, seed=3, class_rows=rows)
    assert_plan_equal(pl, opl)
    sk = pl.new_sketch()
    dW = [to_dev(W, "bf16") for W in Ws]
    usk.build(pl, dW, sk)
    usk.check(pl)
    osk = orc.build_model(opl, Ws)
    np.testing.assert_array_equal(sketch_cells(sk, pl, "bf16"), osk)
    rng = np.random.default_rng(2)
    for l, (o, i) in enumerate(shapes):
        rs = np.sort(rng.choice(o, 6, replace=False))
        Wr = torch.empty((o, i), dtype=torch.bfloat16, device="cuda")
        usk.reconstruct(pl, sk, l, Wr)
        got = w_bits(Wr, "bf16")
        for r in rs:
            np.testing.assert_array_equal(got[r], orc.reconstruct_rows(opl, osk, l, int(r), int(r) + 1)[0])
        x = synth.vector(i, seed=70 + l)[0]
        y = torch.empty(o, dtype=torch.float32, device="cuda")
        usk.linear(pl, sk, l, torch.from_numpy(x).cuda().view(1, -1), y.view(1, -1), usk.new_workspace(pl, l))
        yc = y.cpu().numpy().astype(np.float64)
        for r in rs:
            y64 = orc.linear_rows(opl, osk, l, x.astype(np.float64), int(r), int(r) + 1)[0]
            wv = orc.value_of(got[r], 1)[None, :]
            assert gemv_err(yc[r:r + 1], y64, x.astype(np.float64), wv) <= 1e-5


def test_classrows_prefill(orc, usk):
    """T > 1 (reconstruct + tcgen05 GEMM) on a mixed-rows plan: within the bf16 prefill bar."""
    shapes = [(256, 192)]
    case = (shapes, "bf16", 1.0, (3, 1), "row", 1, 0)
    pl, opl, sk, osk, Ws, dW = _both(orc, usk, case)
    T = 160
    X = synth.torch_vector(192, 5, "cuda", torch.bfloat16, T=T)
    Y = torch.empty((T, 256), dtype=torch.bfloat16, device="cuda")
    usk.linear(pl, sk, 0, X, Y, usk.new_workspace(pl, 0, T))
    x64 = X.float().cpu().numpy().astype(np.float64)
    y64 = orc.linear_rows(opl, osk, 0, x64)
    wv = orc.value_of(orc.reconstruct_rows(opl, osk, 0), 1).reshape(256, 192)
    scale = np.maximum(np.abs(x64) @ np.abs(wv).T, 1e-30)
    assert float(np.max(np.abs(Y.float().cpu().numpy() - y64) / scale)) <= 2e-2


def test_classrows_errors(usk):
    shapes = [(64, 64)]
    for bad in ((0, 1), (9, 2)):
        with pytest.raises(usk.UskError):
            usk.plan_allocation(shapes, bpw=2.0, n_classes=2, class_rows=bad)
    with pytest.raises(usk.UskError):
        usk.plan_allocation(shapes, bpw=2.0, n_classes=2, class_rows=(3, 1), layer_importance=[1.0])
    with pytest.raises(usk.UskError):
        usk.plan_allocation(shapes, bpw=2.0, n_classes=2, class_rows=(3, 1), variant="countmin")
    with pytest.raises(usk.UskError):
        usk.plan_allocation(shapes, bpw=2.0, n_classes=2, class_rows=(3,))   # one count per class
