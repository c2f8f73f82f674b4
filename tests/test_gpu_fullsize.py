"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times.

  c2: one Llama-3.2-1B MLP block, M=3, 0.5 bpw, importance-aware (C=4): every sketch byte and
      the plan arrays vs the oracle; sampled reconstruction rows and GEMV rows.
  c3: all 112 Llama-3.2-1B linears built in ONE usk_build call with the bench's device-generated
      weights; sampled units of sampled layers (sketch bytes + reconstructed entries) and sampled
      GEMV rows of the grouped launches (usk_linear_batch, as timed by bench.py).
  c4: prefill of the 1B gate projection with 2048 x 8 = 16384 tokens at 0.5 and 0.8 bpw
      (reconstruct + tcgen05 GEMM), sampled (token, output) entries vs the fp64 oracle.
  c5: Llama-3-8B-shaped block: plan parity, sampled unit bytes, sampled GEMV rows.
"""
import numpy as np
import pytest

import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

SEED = 0x5EED000000000003


@pytest.fixture(scope="module")
def usk():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2506_17255_b200 import usk as u
    return u


def host_bits(t):
    return t.cpu().view(torch.int16).numpy().view(np.uint16)


def dev_bf16(bits):
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16).copy()).view(torch.bfloat16).cuda()


def gemv_err(y, y64, x64, Wr):
    scale = np.abs(x64)[None, :] @ np.abs(Wr).T
    return float(np.max(np.abs(y - y64) / np.maximum(scale, 1e-30)))


def test_c2_mlp_block_importance(orc, usk):
    shapes = synth.mlp_block_1b_shapes()
    Ws = [synth.weights_bf16(o, i, synth.seed_for(2, 0, 4 + k)) for k, (o, i) in enumerate(shapes)]
    # saliency = Eq. 7 of synthetic calibration activations (oracle fp64 -> fp32, fed to both sides)
    sal = [orc.importance(synth.activations(512, i, seed=200 + k)).astype(np.float32) for k, (o, i) in enumerate(shapes)]
    pl = usk.plan_allocation(shapes, bpw=0.5, rows=3, n_classes=4, seed=SEED,
                             saliency=[torch.from_numpy(s).cuda() for s in sal])
    opl = orc.plan(shapes, 0.5, M=3, dtype=orc.BF16, saliency=sal, C=4, seed=SEED)
    for l in range(3):
        cls, ncols, _, offs = pl.export(l)
        u0, u1 = opl.layer_units(l)
        assert np.array_equal(cls, opl.cls[u0:u1]) and np.array_equal(ncols, opl.ncols[u0:u1])
        assert np.array_equal(offs, opl.offsets[u0:u1 + 1])
        assert pl.layers[l].achieved_bits <= pl.layers[l].budget_bits
    sk = pl.new_sketch()
    usk.build(pl, [dev_bf16(W) for W in Ws], sk)
    usk.check(pl)
    osk = orc.build_model(opl, Ws)
    assert np.array_equal(sk.cpu().numpy().view(np.uint16)[:opl.total_cells], osk)
    rng = np.random.default_rng(0)
    for l, (o, i) in enumerate(shapes):
        Wr = torch.empty((o, i), dtype=torch.bfloat16, device="cuda")
        usk.reconstruct(pl, sk, l, Wr)
        rows = rng.choice(o, 24, replace=False)
        got = host_bits(Wr)[rows]
        for k, r in enumerate(rows):
            assert np.array_equal(got[k], orc.reconstruct_rows(opl, osk, l, int(r), int(r) + 1)[0])
        xb = synth.f32_to_bf16_bits(synth.vector(i, seed=l)[0])
        y = torch.empty(o, dtype=torch.float32, device="cuda")
        usk.linear(pl, sk, l, dev_bf16(xb).view(1, -1), y.view(1, -1), usk.new_workspace(pl, l))
        x64 = synth.bf16_bits_to_f32(xb).astype(np.float64)
        r0 = int(rng.integers(0, o - 16))
        y64 = orc.linear_rows(opl, osk, l, x64, r0, r0 + 16)[0]
        W64 = orc.value_of(orc.reconstruct_rows(opl, osk, l, r0, r0 + 16), orc.BF16).reshape(16, i)
        assert gemv_err(y.cpu().numpy()[r0:r0 + 16].astype(np.float64), y64, x64, W64) <= 1e-5


def _unit_parity(orc, usk, pl, opl, sk, l, W_dev, n_units, rng):
    """Sampled units of layer l: the oracle builds them from the same (device-generated) weights."""
    o, i = opl.shapes[l]
    ts = np.sort(rng.choice(i, n_units, replace=False))
    Wh = np.zeros((o, i), np.uint16)
    cols = host_bits(W_dev[:, torch.from_numpy(ts).cuda()].contiguous())
    Wh[:, ts] = cols
    osk = np.zeros(opl.total_cells, np.uint16)
    for t in ts:
        orc.build_layer(opl, l, Wh, osk, int(t), int(t) + 1)
    u0, _ = opl.layer_units(l)
    got = sk.cpu().numpy().view(np.uint16)
    for t in ts:
        a, b = opl.offsets[u0 + t], opl.offsets[u0 + t + 1]
        assert np.array_equal(got[a:b], osk[a:b]), (l, t)
    # reconstructed entries of those units
    Wr = torch.empty((o, i), dtype=torch.bfloat16, device="cuda")
    usk.reconstruct(pl, sk, l, Wr)
    oj = np.stack([rng.integers(0, o, 256), rng.choice(ts, 256)], 1)
    want = orc.reconstruct_entries(opl, osk, l, oj)
    assert np.array_equal(host_bits(Wr)[oj[:, 0], oj[:, 1]].astype(np.uint32), want)


def test_c3_full_model_sampled(orc, usk):
    shapes = synth.llama32_1b_shapes()
    pl = usk.plan_allocation(shapes, bpw=0.5, rows=3, seed=SEED)
    opl = orc.plan(shapes, 0.5, M=3, dtype=orc.BF16, seed=SEED)
    assert pl.info["total_cells"] == opl.total_cells
    sk = pl.new_sketch()
    ws = [synth.torch_weights_bf16(o, i, synth.seed_for(3, l // 7, l % 7), "cuda") for l, (o, i) in enumerate(shapes)]
    usk.build(pl, ws, sk)  # one call, as bench.py
    usk.check(pl)
    rng = np.random.default_rng(1)
    sample_layers = [0, 1, 3, 4, 6, 7 * 15 + 2, 7 * 15 + 5]
    for l in sample_layers:
        _unit_parity(orc, usk, pl, opl, sk, l, ws[l], 6, rng)
    # grouped GEMV (bench launch configuration) on sampled rows of every group kind (q|k|v, o,
    # gate|up, down; the 8-row-subtile kernel runs q|k|v): the oracle builds the full layers from
    # the same weights
    for g in ([0, 1, 2], [3], [4, 5], [6]):
        i = shapes[g[0]][1]
        x = synth.torch_vector(i, 1000 + g[0], "cuda", torch.bfloat16)[0]
        ys = [torch.empty(shapes[l][0], dtype=torch.float32, device="cuda") for l in g]
        usk.linear_batch(pl, sk, g, x, ys, usk.new_batch_workspace(pl, g))
        x64 = synth.bf16_bits_to_f32(host_bits(x)).astype(np.float64)
        for l, y in zip(g, ys):
            o = shapes[l][0]
            osk = np.zeros(opl.total_cells, np.uint16)
            orc.build_layer(opl, l, host_bits(ws[l]), osk)
            r0 = int(rng.integers(0, o - 8))
            y64 = orc.linear_rows(opl, osk, l, x64, r0, r0 + 8)[0]
            W64 = orc.value_of(orc.reconstruct_rows(opl, osk, l, r0, r0 + 8), orc.BF16).reshape(8, i)
            assert gemv_err(y.cpu().numpy()[r0:r0 + 8].astype(np.float64), y64, x64, W64) <= 1e-5


@pytest.mark.parametrize("bpw,k", [(0.5, 4), (0.8, 4), (0.5, 6), (0.5, 1)], ids=["gate-0.5", "gate-0.8", "down-0.5",
                                                                                 "k-0.5"])
def test_c4_prefill_16384_tokens(orc, usk, bpw, k):
    # every distinct GEMM geometry the config-4 bench pass times: gate/up [8192, 2048], down
    # [2048, 8192] (K = 8192: 128 K-blocks), k/v [512, 2048] (N = 512); q/o share gate's K
    o, i = synth.llama_block(2048, 512, 8192)[k]
    T = 16384
    W = synth.torch_weights_bf16(o, i, synth.seed_for(4, 0, k), "cuda")
    pl = usk.plan_allocation([(o, i)], bpw=bpw, rows=3, seed=SEED)
    opl = orc.plan([(o, i)], bpw, M=3, dtype=orc.BF16, seed=SEED)
    sk = pl.new_sketch()
    usk.build(pl, [W], sk)
    X = synth.torch_vector(i, 7, "cuda", torch.bfloat16, T=T)
    Y = torch.empty((T, o), dtype=torch.bfloat16, device="cuda")
    usk.linear(pl, sk, 0, X, Y, usk.new_workspace(pl, 0, T))
    osk = np.zeros(opl.total_cells, np.uint16)
    orc.build_layer(opl, 0, host_bits(W), osk)
    rng = np.random.default_rng(2)
    rows = rng.choice(o, 8, replace=False)
    toks = rng.choice(T, 64, replace=False)
    Xh = synth.bf16_bits_to_f32(host_bits(X[torch.from_numpy(toks).cuda()])).astype(np.float64)
    Yh = Y.float().cpu().numpy()
    for r in rows:
        y64 = orc.linear_rows(opl, osk, 0, Xh, int(r), int(r) + 1)[:, 0]
        w64 = orc.value_of(orc.reconstruct_rows(opl, osk, 0, int(r), int(r) + 1), orc.BF16).reshape(i)
        scale = np.abs(Xh) @ np.abs(w64)
        err = np.max(np.abs(Yh[toks, r] - y64) / np.maximum(scale, 1e-30))
        assert err <= 2e-2, err


def test_c5_llama8b_block(orc, usk):
    shapes = synth.llama3_8b_shapes()[:7]
    pl = usk.plan_allocation(shapes, bpw=0.5, rows=3, seed=SEED)
    opl = orc.plan(shapes, 0.5, M=3, dtype=orc.BF16, seed=SEED)
    for l in range(7):
        _, ncols, _, offs = pl.export(l)
        u0, u1 = opl.layer_units(l)
        assert np.array_equal(ncols, opl.ncols[u0:u1]) and np.array_equal(offs, opl.offsets[u0:u1 + 1])
    sk = pl.new_sketch()
    ws = [synth.torch_weights_bf16(o, i, synth.seed_for(5, 0, l), "cuda") for l, (o, i) in enumerate(shapes)]
    usk.build(pl, ws, sk)
    usk.check(pl)
    rng = np.random.default_rng(3)
    for l in (0, 4, 6):
        _unit_parity(orc, usk, pl, opl, sk, l, ws[l], 4, rng)
    l = 6  # down [4096, 14336]
    o, i = shapes[l]
    x = synth.torch_vector(i, 11, "cuda", torch.bfloat16)
    y = torch.empty((1, o), dtype=torch.float32, device="cuda")
    usk.linear(pl, sk, l, x, y, usk.new_workspace(pl, l))
    osk = np.zeros(opl.total_cells, np.uint16)
    orc.build_layer(opl, l, host_bits(ws[l]), osk)
    x64 = synth.bf16_bits_to_f32(host_bits(x)[0]).astype(np.float64)
    r0 = 1000
    y64 = orc.linear_rows(opl, osk, l, x64, r0, r0 + 8)[0]
    W64 = orc.value_of(orc.reconstruct_rows(opl, osk, l, r0, r0 + 8), orc.BF16).reshape(8, i)
    assert gemv_err(y.cpu().numpy()[0, r0:r0 + 8].astype(np.float64), y64, x64, W64) <= 1e-5


def test_q4_gemv_gate_up_batch(orc, usk):
    # the paper's 0.5-bpw point (q4 states, G = 128; bench.py paper_point_q4) at the Llama-3.2-1B
    # gate|up geometry through usk_linear_batch, the launch the bench times (UPL = 1 slots)
    shapes = [(8192, 2048), (8192, 2048)]
    pl = usk.plan_allocation(shapes, bpw=0.5, rows=3, seed=SEED, state_bits=4, group_size=128)
    opl = orc.plan(shapes, 0.5, M=3, dtype=orc.BF16, seed=SEED, state_bits=4, group=128)
    ws = [synth.torch_weights_bf16(o, i, synth.seed_for(3, 0, 4 + l), "cuda") for l, (o, i) in enumerate(shapes)]
    sk = pl.new_sketch()
    usk.build(pl, ws, sk)
    usk.check(pl)
    osk = orc.build_model(opl, [host_bits(w) for w in ws])
    nb = pl.info["total_cells"] * 4 // 8
    assert np.array_equal(sk.cpu().numpy()[:nb], osk.packed)
    x = synth.torch_vector(2048, 1004, "cuda", torch.bfloat16)[0]
    ys = [torch.empty(8192, dtype=torch.float32, device="cuda") for _ in shapes]
    usk.linear_batch(pl, sk, [0, 1], x, ys, usk.new_batch_workspace(pl, [0, 1]))
    x64 = synth.bf16_bits_to_f32(host_bits(x)).astype(np.float64)
    rng = np.random.default_rng(8)
    for l, y in enumerate(ys):
        r0 = int(rng.integers(0, 8192 - 8))
        y64 = orc.linear_rows(opl, osk, l, x64, r0, r0 + 8)[0]
        Wdq = orc.linear_rows(opl, osk, l, np.eye(2048), r0, r0 + 8).T  # fp32-dequantised W' rows
        assert gemv_err(y.cpu().numpy()[r0:r0 + 8].astype(np.float64), y64, x64, Wdq) <= 1e-5


def _query_units(orc, usk, pl, opl, sk, l, W_dev, n_units, rng):
    """Query layout: sampled units of layer l rebuilt by the oracle from the same weights, compared
    with the units read back from the GPU query bytes (tests/qlayout.py, from usk.h's text)."""
    import qlayout
    o, i = opl.shapes[l]
    ts = np.sort(rng.choice(i, n_units, replace=False))
    Wh = np.zeros((o, i), np.uint16)
    Wh[:, ts] = host_bits(W_dev[:, torch.from_numpy(ts).cuda()].contiguous())
    osk = np.zeros(opl.total_cells, np.uint16)
    for t in ts:
        orc.build_layer(opl, l, Wh, osk, int(t), int(t) + 1)
    u0, u1 = opl.layer_units(l)
    li = pl.layers[l]
    q = sk.cpu().numpy().view(np.uint16)[li.qbyte_begin // 2:(li.qbyte_begin + li.qbytes) // 2]
    for t in ts:
        a, b = opl.offsets[u0 + t], opl.offsets[u0 + t + 1]
        got = qlayout.unit_cells(q, opl.ncols[u0:u1], opl.nrows[u0:u1], int(t), opl.M)
        assert np.array_equal(got, osk[a:b]), (l, t)
    Wr = torch.empty((o, i), dtype=torch.bfloat16, device="cuda")
    usk.reconstruct(pl, sk, l, Wr)
    oj = np.stack([rng.integers(0, o, 256), rng.choice(ts, 256)], 1)
    assert np.array_equal(host_bits(Wr)[oj[:, 0], oj[:, 1]].astype(np.uint32), orc.reconstruct_entries(opl, osk, l, oj))


def test_c3_query_layout_full_model_sampled(orc, usk):
    """The bench's headline plan: USK-XG keys in the query layout (ledger L32), all 112 linears built
    in one call; sampled units + reconstructed entries, and sampled rows of every grouped GEMV kind."""
    shapes = synth.llama32_1b_shapes()
    pl = usk.plan_allocation(shapes, bpw=0.5, rows=3, seed=SEED, hash="xg", layout="query")
    opl = orc.plan(shapes, 0.5, M=3, dtype=orc.BF16, seed=SEED, hash_kind=orc.HASH_XG)
    assert pl.info["total_cells"] == opl.total_cells
    sk = pl.new_sketch()
    ws = [synth.torch_weights_bf16(o, i, synth.seed_for(3, l // 7, l % 7), "cuda") for l, (o, i) in enumerate(shapes)]
    usk.build(pl, ws, sk)
    usk.check(pl)
    rng = np.random.default_rng(11)
    for l in [0, 1, 3, 4, 6, 7 * 15 + 2, 7 * 15 + 5]:
        _query_units(orc, usk, pl, opl, sk, l, ws[l], 6, rng)
    for g in ([0, 1, 2], [3], [4, 5], [6], [7 * 15 + 4, 7 * 15 + 5]):
        i = shapes[g[0]][1]
        x = synth.torch_vector(i, 1000 + g[0], "cuda", torch.bfloat16)[0]
        ys = [torch.empty(shapes[l][0], dtype=torch.float32, device="cuda") for l in g]
        usk.linear_batch(pl, sk, g, x, ys, usk.new_batch_workspace(pl, g))
        x64 = synth.bf16_bits_to_f32(host_bits(x)).astype(np.float64)
        for l, y in zip(g, ys):
            o = shapes[l][0]
            osk = np.zeros(opl.total_cells, np.uint16)
            orc.build_layer(opl, l, host_bits(ws[l]), osk)
            for r0 in (0, int(rng.integers(0, o - 8)), o - 8):
                y64 = orc.linear_rows(opl, osk, l, x64, r0, r0 + 8)[0]
                W64 = orc.value_of(orc.reconstruct_rows(opl, osk, l, r0, r0 + 8), orc.BF16).reshape(8, i)
                assert gemv_err(y.cpu().numpy()[r0:r0 + 8].astype(np.float64), y64, x64, W64) <= 1e-5


def test_c3_xg_importance_classes_full_model(orc, usk):
    """The bench's importance point at full size: C = 4 saliency classes scored per key group (ledger
    L33) with class rows (3, 3, 2, 2) (L30), USK-XG keys, all 112 linears, unit-major layout (the
    grouped-key build K2).  The whole plan (class, N, M of every unit) equals the oracle's; sampled
    units, reconstructed entries and grouped GEMV rows.  (The query layout of the same plan:
    test_c3_query_importance_classes_full_model.)"""
    shapes = synth.llama32_1b_shapes()
    sal = [synth.saliency_like(i, 500 + l) for l, (o, i) in enumerate(shapes)]
    crows = (3, 3, 2, 2)
    sal_dev = [torch.from_numpy(s).cuda() for s in sal]
    pl = usk.plan_allocation(shapes, bpw=0.5, rows=3, seed=SEED, hash="xg", n_classes=4, saliency=sal_dev,
                             class_rows=crows)
    opl = orc.plan(shapes, 0.5, M=3, dtype=orc.BF16, seed=SEED, hash_kind=orc.HASH_XG, saliency=sal, C=4,
                   class_rows=crows)
    assert pl.info["total_cells"] == opl.total_cells
    for l in range(len(shapes)):
        cls, ncols, nrows, offs = pl.export(l)
        u0, u1 = opl.layer_units(l)
        np.testing.assert_array_equal(cls, opl.cls[u0:u1])
        np.testing.assert_array_equal(ncols, opl.ncols[u0:u1])
        np.testing.assert_array_equal(nrows, opl.nrows[u0:u1])
        assert (ncols.reshape(-1, 8) == ncols.reshape(-1, 8)[:, :1]).all()
    sk = pl.new_sketch()
    ws = [synth.torch_weights_bf16(o, i, synth.seed_for(3, l // 7, l % 7), "cuda") for l, (o, i) in enumerate(shapes)]
    usk.build(pl, ws, sk)
    usk.check(pl)
    rng = np.random.default_rng(12)
    for l in [0, 4, 6, 7 * 9 + 1]:
        _unit_parity(orc, usk, pl, opl, sk, l, ws[l], 8, rng)
    for g in ([0, 1, 2], [4, 5], [6]):
        i = shapes[g[0]][1]
        x = synth.torch_vector(i, 2000 + g[0], "cuda", torch.bfloat16)[0]
        ys = [torch.empty(shapes[l][0], dtype=torch.float32, device="cuda") for l in g]
        usk.linear_batch(pl, sk, g, x, ys, usk.new_batch_workspace(pl, g))
        x64 = synth.bf16_bits_to_f32(host_bits(x)).astype(np.float64)
        for l, y in zip(g, ys):
            o = shapes[l][0]
            osk = np.zeros(opl.total_cells, np.uint16)
            orc.build_layer(opl, l, host_bits(ws[l]), osk)
            for r0 in (0, int(rng.integers(0, o - 8)), o - 8):
                y64 = orc.linear_rows(opl, osk, l, x64, r0, r0 + 8)[0]
                W64 = orc.value_of(orc.reconstruct_rows(opl, osk, l, r0, r0 + 8), orc.BF16).reshape(8, i)
                assert gemv_err(y.cpu().numpy()[r0:r0 + 8].astype(np.float64), y64, x64, W64) <= 1e-5


def test_c3_query_importance_classes_full_model(orc, usk):
    """The bench's importance point in the query layout (ledger L34): key groups in class order, the
    most salient class of gate/up (N ~ 300 at 3 rows) in 64-unit chunks, the others in 256-unit
    chunks; bytes of all layers = the unit-major bytes (no padding).  Sampled units (read back with
    tests/qlayout.py from usk.h's text), reconstructed entries and grouped GEMV rows vs the oracle."""
    import qlayout
    shapes = synth.llama32_1b_shapes()
    sal = [synth.saliency_like(i, 500 + l) for l, (o, i) in enumerate(shapes)]
    crows = (3, 3, 2, 2)
    pl = usk.plan_allocation(shapes, bpw=0.5, rows=3, seed=SEED, hash="xg", layout="query", n_classes=4,
                             saliency=[torch.from_numpy(s).cuda() for s in sal], class_rows=crows)
    opl = orc.plan(shapes, 0.5, M=3, dtype=orc.BF16, seed=SEED, hash_kind=orc.HASH_XG, saliency=sal, C=4,
                   class_rows=crows)
    assert pl.sketch_bytes <= 2 * opl.total_cells + 512 * 112 * 64  # class-cut chunks: a few partial slots
    sk = pl.new_sketch()
    ws = [synth.torch_weights_bf16(o, i, synth.seed_for(3, l // 7, l % 7), "cuda") for l, (o, i) in enumerate(shapes)]
    usk.build(pl, ws, sk)
    usk.check(pl)
    rng = np.random.default_rng(13)
    q = sk.cpu().numpy().view(np.uint16)
    for l in [0, 1, 4, 5, 6, 7 * 9 + 4]:
        o, i = shapes[l]
        u0, u1 = opl.layer_units(l)
        li = pl.layers[l]
        qb = q[li.qbyte_begin // 2:(li.qbyte_begin + li.qbytes) // 2]
        ts = np.sort(rng.choice(i, 6, replace=False))
        Wh = np.zeros((o, i), np.uint16)
        Wh[:, ts] = host_bits(ws[l][:, torch.from_numpy(ts).cuda()].contiguous())
        osk = np.zeros(opl.total_cells, np.uint16)
        for t in ts:
            orc.build_layer(opl, l, Wh, osk, int(t), int(t) + 1)
            a, b = opl.offsets[u0 + t], opl.offsets[u0 + t + 1]
            got = qlayout.unit_cells(qb, opl.ncols[u0:u1], opl.nrows[u0:u1], int(t), 3, opl.cls[u0:u1])
            assert np.array_equal(got, osk[a:b]), (l, t)
        Wr = torch.empty((o, i), dtype=torch.bfloat16, device="cuda")
        usk.reconstruct(pl, sk, l, Wr)
        oj = np.stack([rng.integers(0, o, 128), rng.choice(ts, 128)], 1)
        assert np.array_equal(host_bits(Wr)[oj[:, 0], oj[:, 1]].astype(np.uint32), orc.reconstruct_entries(opl, osk, l, oj))
    for g in ([0, 1, 2], [4, 5], [6]):
        i = shapes[g[0]][1]
        x = synth.torch_vector(i, 3000 + g[0], "cuda", torch.bfloat16)[0]
        ys = [torch.empty(shapes[l][0], dtype=torch.float32, device="cuda") for l in g]
        usk.linear_batch(pl, sk, g, x, ys, usk.new_batch_workspace(pl, g))
        x64 = synth.bf16_bits_to_f32(host_bits(x)).astype(np.float64)
        for l, y in zip(g, ys):
            o = shapes[l][0]
            osk = np.zeros(opl.total_cells, np.uint16)
            orc.build_layer(opl, l, host_bits(ws[l]), osk)
            for r0 in (0, int(rng.integers(0, o - 8)), o - 8):
                y64 = orc.linear_rows(opl, osk, l, x64, r0, r0 + 8)[0]
                W64 = orc.value_of(orc.reconstruct_rows(opl, osk, l, r0, r0 + 8), orc.BF16).reshape(8, i)
                assert gemv_err(y.cpu().numpy()[r0:r0 + 8].astype(np.float64), y64, x64, W64) <= 1e-5


@pytest.mark.parametrize("k", [4, 6, 1], ids=["gate", "down", "k"])
def test_c4_query_prefill_16384_tokens(orc, usk, k):
    """Config 4 on the query layout (K3p into the workspace + the tcgen05 GEMM), T = 16384."""
    o, i = synth.llama_block(2048, 512, 8192)[k]
    T = 16384
    W = synth.torch_weights_bf16(o, i, synth.seed_for(4, 0, k), "cuda")
    pl = usk.plan_allocation([(o, i)], bpw=0.5, rows=3, seed=SEED, hash="xg", layout="query")
    opl = orc.plan([(o, i)], 0.5, M=3, dtype=orc.BF16, seed=SEED, hash_kind=orc.HASH_XG)
    sk = pl.new_sketch()
    usk.build(pl, [W], sk)
    X = synth.torch_vector(i, 7, "cuda", torch.bfloat16, T=T)
    Y = torch.empty((T, o), dtype=torch.bfloat16, device="cuda")
    usk.linear(pl, sk, 0, X, Y, usk.new_workspace(pl, 0, T))
    osk = np.zeros(opl.total_cells, np.uint16)
    orc.build_layer(opl, 0, host_bits(W), osk)
    rng = np.random.default_rng(5)
    toks = rng.choice(T, 64, replace=False)
    Xh = synth.bf16_bits_to_f32(host_bits(X[torch.from_numpy(toks).cuda()])).astype(np.float64)
    Yh = Y.float().cpu().numpy()
    for r in rng.choice(o, 8, replace=False):
        y64 = orc.linear_rows(opl, osk, 0, Xh, int(r), int(r) + 1)[:, 0]
        w64 = orc.value_of(orc.reconstruct_rows(opl, osk, 0, int(r), int(r) + 1), orc.BF16).reshape(i)
        err = np.max(np.abs(Yh[toks, r] - y64) / np.maximum(np.abs(Xh) @ np.abs(w64), 1e-30))
        assert err <= 2e-2, err


def test_c5_query_llama8b_block(orc, usk):
    """Llama-3-8B block on the query layout: gate/up ([14336, 4096], N = 149 at 0.5 bpw: a 256-unit
    chunk would take 229 KB) use 128-unit chunks (usk.h), the others 256; the 14336-wide down has 56
    chunks.  Sampled units and rows of q, gate and down."""
    shapes = synth.llama3_8b_shapes()[:7]
    pl = usk.plan_allocation(shapes, bpw=0.5, rows=3, seed=SEED, hash="xg", layout="query")
    assert [pl.layers[l].qchunk_units for l in range(7)] == [256, 256, 256, 256, 128, 128, 256]
    opl = orc.plan(shapes, 0.5, M=3, dtype=orc.BF16, seed=SEED, hash_kind=orc.HASH_XG)
    sk = pl.new_sketch()
    ws = [synth.torch_weights_bf16(o, i, synth.seed_for(5, 0, l), "cuda") for l, (o, i) in enumerate(shapes)]
    usk.build(pl, ws, sk)
    usk.check(pl)
    rng = np.random.default_rng(13)
    for l in (0, 4, 6):
        _query_units(orc, usk, pl, opl, sk, l, ws[l], 4, rng)
    g = [4, 5]  # gate|up: the 128-unit chunk kernels, one grouped call
    x = synth.torch_vector(4096, 12, "cuda", torch.bfloat16)[0]
    ys = [torch.empty(14336, dtype=torch.float32, device="cuda") for _ in g]
    usk.linear_batch(pl, sk, g, x, ys, usk.new_batch_workspace(pl, g))
    x64 = synth.bf16_bits_to_f32(host_bits(x)).astype(np.float64)
    for l, yv in zip(g, ys):
        osk = np.zeros(opl.total_cells, np.uint16)
        orc.build_layer(opl, l, host_bits(ws[l]), osk)
        for r0 in (0, 7000, 14336 - 8):
            y64 = orc.linear_rows(opl, osk, l, x64, r0, r0 + 8)[0]
            W64 = orc.value_of(orc.reconstruct_rows(opl, osk, l, r0, r0 + 8), orc.BF16).reshape(8, 4096)
            assert gemv_err(yv.cpu().numpy()[r0:r0 + 8].astype(np.float64), y64, x64, W64) <= 1e-5
    l = 6
    o, i = shapes[l]
    x = synth.torch_vector(i, 11, "cuda", torch.bfloat16)
    y = torch.empty((1, o), dtype=torch.float32, device="cuda")
    usk.linear(pl, sk, l, x, y, usk.new_workspace(pl, l))
    osk = np.zeros(opl.total_cells, np.uint16)
    orc.build_layer(opl, l, host_bits(ws[l]), osk)
    x64 = synth.bf16_bits_to_f32(host_bits(x)[0]).astype(np.float64)
    y64 = orc.linear_rows(opl, osk, l, x64, 1000, 1008)[0]
    W64 = orc.value_of(orc.reconstruct_rows(opl, osk, l, 1000, 1008), orc.BF16).reshape(8, i)
    assert gemv_err(y.cpu().numpy()[0, 1000:1008].astype(np.float64), y64, x64, W64) <= 1e-5


def test_c4_batch_tokens_groups_16384_tokens(orc, usk):
    """Config 4 as the bench runs it: q|k|v and gate|up of a Llama-3.2-1B block through
    usk_linear_batch_tokens at T = 16384 (one batched reconstruction + one GEMM per group) equal the
    per-layer usk_linear results bit for bit; sampled entries within 2e-2 of the oracle."""
    shapes = synth.llama_block(2048, 512, 8192)
    T = 16384
    pl = usk.plan_allocation(shapes, bpw=0.5, rows=3, seed=SEED, hash="xg", layout="query")
    opl = orc.plan(shapes, 0.5, M=3, dtype=orc.BF16, seed=SEED, hash_kind=orc.HASH_XG)
    ws = [synth.torch_weights_bf16(o, i, synth.seed_for(4, 0, k), "cuda") for k, (o, i) in enumerate(shapes)]
    sk = pl.new_sketch()
    usk.build(pl, ws, sk)
    X = synth.torch_vector(2048, 8, "cuda", torch.bfloat16, T=T)
    rng = np.random.default_rng(6)
    toks = rng.choice(T, 32, replace=False)
    Xh = synth.bf16_bits_to_f32(host_bits(X[torch.from_numpy(toks).cuda()])).astype(np.float64)
    for g in ([0, 1, 2], [4, 5]):
        ys = [torch.empty((T, shapes[l][0]), dtype=torch.bfloat16, device="cuda") for l in g]
        wsp = torch.zeros(usk.linear_batch_tokens_workspace_bytes(pl, g, T), dtype=torch.uint8, device="cuda")
        usk.linear_batch_tokens(pl, sk, g, X, ys, wsp)
        for l, y in zip(g, ys):
            o = shapes[l][0]
            ref = torch.empty((T, o), dtype=torch.bfloat16, device="cuda")
            usk.linear(pl, sk, l, X, ref, usk.new_workspace(pl, l, T))
            assert torch.equal(y, ref), l
            osk = np.zeros(opl.total_cells, np.uint16)
            orc.build_layer(opl, l, host_bits(ws[l]), osk)
            Yh = y.float().cpu().numpy()
            for r in rng.choice(o, 4, replace=False):
                y64 = orc.linear_rows(opl, osk, l, Xh, int(r), int(r) + 1)[:, 0]
                w64 = orc.value_of(orc.reconstruct_rows(opl, osk, l, int(r), int(r) + 1), orc.BF16).reshape(-1)
                err = np.max(np.abs(Yh[toks, r] - y64) / np.maximum(np.abs(Xh) @ np.abs(w64), 1e-30))
                assert err <= 2e-2, err
