"""GPU parity of the query layout (usk.h USK_LAYOUT_QUERY, USK-XG keys; DESIGN.md ledger L32) through
the C ABI against the CPU oracle on the same seeded inputs:

* sketch bytes: the GPU query sketch, unpacked with tests/qlayout.py (written from usk.h's text), equals
  the oracle's unit-major sketch bit for bit, and every padding word is 0;
* reconstruction (K3p) bit-exact, any row range and leading dimension;
* sketch-GEMV (K4p) within max_o |y - y64| / sum_j |x_j w'_oj| <= 1e-5 of the oracle's fp64 result for
  bf16 and fp32 x, fp32 and bf16 y; deterministic; output shards and batched calls bit-identical to
  the single full call."""
import numpy as np
import pytest

import synth
import qlayout  # tests/qlayout.py (pytest puts tests/ on sys.path)

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def usk():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2506_17255_b200 import usk as u
    return u


def to_dev(W):
    return torch.from_numpy(W.view(np.int16).copy()).view(torch.bfloat16).cuda()


def gemv_err(y, y64, x, Wr):
    scale = np.maximum(np.abs(x)[None, :] @ np.abs(Wr).T, 1e-30)
    return float(np.max(np.abs(y - y64) / scale))


def build_both(orc, usk, shapes, bpw=0.5, M=3, seed=77, wseed=5, kind=None, saliency=None, C=None):
    Ws = []
    for k, (o, i) in enumerate(shapes):
        Ws.append(synth.edge_matrix_bf16(kind, o, i, wseed + k) if kind else synth.weights_bf16(o, i, wseed + k))
    sal_dev = None if saliency is None else [torch.from_numpy(s).cuda() for s in saliency]
    pl = usk.plan_allocation(shapes, bpw=bpw, rows=M, hash="xg", layout="query", seed=seed, saliency=sal_dev,
                             n_classes=0 if C is None else C)
    opl = orc.plan(shapes, bpw, M=M, dtype=orc.BF16, hash_kind=orc.HASH_XG, seed=seed, saliency=saliency, C=C)
    sk = pl.new_sketch()
    sk.fill_(0xCD)
    usk.build(pl, [to_dev(W) for W in Ws], sk)
    usk.check(pl)
    osk = orc.build_model(opl, Ws)
    return pl, opl, sk, osk, Ws


SHAPES = [
    [(256, 512), (96, 512)],                # whole chunks; rows not a multiple of 16
    [(200, 72), (49, 72)],                  # one partial chunk (9 key groups)
    [(130, 264)],                           # a full chunk + a 1-group chunk
    [(2048, 512), (512, 512), (8192, 256)], # Llama-like N = 21, 5, 85
    [(8192, 264), (96, 264)],               # N = 170: 128-unit chunks (ld.shared.v2 kernels)
]
BPW = {0: 0.5, 1: 1.0, 2: 0.5, 3: 0.5, 4: 1.0}


@pytest.mark.parametrize("shapes", SHAPES, ids=[str(s[0]) for s in SHAPES])
def test_query_sketch_bytes_and_reconstruct(orc, usk, shapes):
    pl, opl, sk, osk, Ws = build_both(orc, usk, shapes, bpw=BPW[SHAPES.index(shapes)])
    q = sk.cpu().numpy().view(np.uint16)
    offs, total = qlayout.model_offsets([opl.ncols[slice(*opl.layer_units(l))] for l in range(len(shapes))], 3)
    assert pl.info["layout"] == 1 and pl.info["hash"] == 2
    for l, (o, i) in enumerate(shapes):
        u0, u1 = opl.layer_units(l)
        li = pl.layers[l]
        assert li.qbyte_begin == offs[l]
        qb = q[li.qbyte_begin // 2:(li.qbyte_begin + li.qbytes) // 2]
        cells, pad_ok = qlayout.unpack_layer(qb, opl.offsets[u0:u1 + 1], opl.ncols[u0:u1], opl.nrows[u0:u1], 3)
        np.testing.assert_array_equal(cells, osk[opl.offsets[u0]:opl.offsets[u1]])
        assert pad_ok
        # reconstruction: full, a ragged row range, and an odd leading dimension
        w = torch.empty(o, i, dtype=torch.bfloat16, device="cuda")
        usk.reconstruct(pl, sk, l, w)
        ref = orc.reconstruct_rows(opl, osk, l)
        np.testing.assert_array_equal(w.cpu().view(torch.int16).numpy().view(np.uint16).reshape(-1), ref.reshape(-1))
        r0, r1 = min(3, o - 1), o
        buf = torch.zeros(r1 - r0, i + 3, dtype=torch.bfloat16, device="cuda")
        usk.reconstruct(pl, sk, l, buf, r0, r1)
        got = buf[:, :i].cpu().view(torch.int16).numpy().view(np.uint16)
        np.testing.assert_array_equal(got.reshape(-1), orc.reconstruct_rows(opl, osk, l, r0, r1).reshape(-1))
    assert total + 256 <= pl.sketch_bytes


@pytest.mark.parametrize("kind", ["pm_pairs", "zeros", "subnormal", "all_equal", "mixed", "outlier"])
def test_query_edge_values(orc, usk, kind):
    shapes = [(64, 256), (40, 64)]
    pl, opl, sk, osk, Ws = build_both(orc, usk, shapes, bpw=4.0, kind=kind)
    for l, (o, i) in enumerate(shapes):
        w = torch.empty(o, i, dtype=torch.bfloat16, device="cuda")
        usk.reconstruct(pl, sk, l, w)
        np.testing.assert_array_equal(w.cpu().view(torch.int16).numpy().view(np.uint16).reshape(-1),
                                      orc.reconstruct_rows(opl, osk, l).reshape(-1))


@pytest.mark.parametrize("shapes", SHAPES, ids=[str(s[0]) for s in SHAPES])
def test_query_gemv(orc, usk, shapes):
    pl, opl, sk, osk, Ws = build_both(orc, usk, shapes, bpw=BPW[SHAPES.index(shapes)])
    for l, (o, i) in enumerate(shapes):
        Wr = orc.value_of(orc.reconstruct_rows(opl, osk, l), orc.BF16).reshape(o, i)
        for xdt in ("bf16", "f32"):
            x = synth.vector(i, seed=l + 11)[0]
            if xdt == "bf16":
                xb = synth.f32_to_bf16_bits(x)
                xd = torch.from_numpy(xb.view(np.int16).copy()).view(torch.bfloat16).cuda()
                x64 = synth.bf16_bits_to_f32(xb).astype(np.float64)
            else:
                xd = torch.from_numpy(x).cuda()
                x64 = x.astype(np.float64)
            y64 = orc.linear_rows(opl, osk, l, x64)[0]
            ws = usk.new_workspace(pl, l)
            y = torch.empty(o, dtype=torch.float32, device="cuda")
            usk.linear(pl, sk, l, xd.view(1, -1), y.view(1, -1), ws)
            assert gemv_err(y.cpu().numpy().astype(np.float64), y64, x64, Wr) <= 1e-5
            y2 = torch.empty_like(y)
            usk.linear(pl, sk, l, xd.view(1, -1), y2.view(1, -1), ws)
            assert torch.equal(y, y2)
            yb = torch.empty(o, dtype=torch.bfloat16, device="cuda")
            usk.linear(pl, sk, l, xd.view(1, -1), yb.view(1, -1), ws)
            assert torch.equal(yb, y.to(torch.bfloat16))  # RNE of the same fp32 sum
            for h, e in ((o // 2, o), (o // 3 + 1, o - 5), (7, min(o, 47))):
                if e <= h:
                    continue
                ys = torch.empty(e - h, dtype=torch.float32, device="cuda")
                usk.linear(pl, sk, l, xd.view(1, -1), ys.view(1, -1), usk.new_workspace(pl, l, 1, h, e), h, e)
                assert torch.equal(ys, y[h:e]), (h, e)
    # all layers of a shape group that share in_features in one call == single calls
    by_in = {}
    for l, (o, i) in enumerate(shapes):
        by_in.setdefault(i, []).append(l)
    for i, layers in by_in.items():
        xb = synth.f32_to_bf16_bits(synth.vector(i, seed=3)[0])
        xd = torch.from_numpy(xb.view(np.int16).copy()).view(torch.bfloat16).cuda()
        ys = [torch.empty(shapes[l][0], dtype=torch.float32, device="cuda") for l in layers]
        usk.linear_batch(pl, sk, layers, xd, ys, usk.new_batch_workspace(pl, layers))
        for k, l in enumerate(layers):
            y1 = torch.empty(shapes[l][0], dtype=torch.float32, device="cuda")
            usk.linear(pl, sk, l, xd.view(1, -1), y1.view(1, -1), usk.new_workspace(pl, l))
            assert torch.equal(ys[k], y1)


def test_query_prefill(orc, usk):
    """T > 1 on the query layout: K3p into the workspace + the tcgen05 GEMM, within the bf16
    tensor-core tolerance (2e-2 of the fp64 result, scaled as for the GEMV)."""
    shapes = [(384, 512)]
    pl, opl, sk, osk, Ws = build_both(orc, usk, shapes)
    T = 300
    X = synth.weights_bf16(T, 512, 99)
    Xd = to_dev(X)
    Y = torch.empty(T, 384, dtype=torch.float32, device="cuda")
    usk.linear(pl, sk, 0, Xd, Y, usk.new_workspace(pl, 0, T))
    Wr = orc.value_of(orc.reconstruct_rows(opl, osk, 0), orc.BF16).reshape(384, 512)
    X64 = synth.bf16_bits_to_f32(X).astype(np.float64).reshape(T, 512)
    ref = X64 @ Wr.T
    scale = np.maximum(np.abs(X64) @ np.abs(Wr).T, 1e-30)
    assert float(np.max(np.abs(Y.cpu().numpy() - ref) / scale)) <= 2e-2


def test_query_build_paths_agree(usk):
    """The fused K2 write-out (default) and the unit-major build + k_qpack (USK_QBUILD_PACK=1, the
    fallback) write the same query bytes; run in a child process so the env switch takes effect."""
    import os, subprocess, sys
    code = (
        "import sys, hashlib, torch; sys.path.insert(0, %r); import synth; "
        "from paper_2506_17255_b200 import usk; "
        "sh=[(2048,512),(512,512),(200,72)]; "
        "pl=usk.plan_allocation(sh, bpw=0.5, hash='xg', layout='query', seed=9); sk=pl.new_sketch(); sk.zero_(); "
        "ws=[synth.torch_weights_bf16(o,i,30+k,'cuda') for k,(o,i) in enumerate(sh)]; usk.build(pl, ws, sk); usk.check(pl); "
        "print(hashlib.sha256(sk.cpu().numpy().tobytes()).hexdigest())") % os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = []
    for flag in ("0", "1"):
        env = dict(os.environ, USK_QBUILD_PACK=flag)
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr
        out.append(r.stdout.strip().splitlines()[-1])
    assert out[0] == out[1]


def test_query_layout_rejections(usk):
    with pytest.raises(usk.UskError) as e:
        usk.plan_allocation([(64, 64)], bpw=1.0, layout="query")  # USK-X keys
    assert e.value.status == usk.EUNSUPPORTED
    with pytest.raises(usk.UskError) as e:
        usk.plan_allocation([(64, 60)], bpw=1.0, hash="xg", layout="query")  # in % 8
    assert e.value.status == usk.EUNSUPPORTED
    with pytest.raises(usk.UskError) as e:
        usk.plan_allocation([(64, 64)], bpw=1.0, hash="xg", layout="query", dtype="f32")
    assert e.value.status == usk.EUNSUPPORTED
    with pytest.raises(usk.UskError) as e:  # a 256-unit chunk (3 x 833 columns) exceeds shared memory
        usk.plan_allocation([(40000, 16)], bpw=1.0, hash="xg", layout="query")
    assert e.value.status == usk.EUNSUPPORTED
    pl = usk.plan_allocation([(64, 64)], bpw=1.0, hash="xg", layout="query")
    W = torch.zeros(64, 64, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(usk.UskError) as e:
        usk.stats(pl, pl.new_sketch(), 0, W)
    assert e.value.status == usk.EUNSUPPORTED


@pytest.mark.parametrize("shapes,bpw,M", [([(256, 512), (96, 512)], 0.5, 3), ([(200, 72), (49, 72)], 1.0, 3),
                                          ([(130, 264), (2048, 64)], 1.0, 2), ([(512, 40)], 2.0, 1)],
                         ids=["block", "ragged", "M2", "M1"])
def test_xg_unit_major_build_bit_exact(orc, usk, shapes, bpw, M):
    """USK-XG plans in the unit-major layout build with the grouped-key K2 (one shared address per key
    group and sketch row): every sketch byte equals the oracle's, reconstruction and GEMV as usual."""
    Ws = [synth.weights_bf16(o, i, 60 + k) for k, (o, i) in enumerate(shapes)]
    pl = usk.plan_allocation(shapes, bpw=bpw, rows=M, hash="xg", seed=31)
    opl = orc.plan(shapes, bpw, M=M, dtype=orc.BF16, hash_kind=orc.HASH_XG, seed=31)
    sk = pl.new_sketch()
    sk.fill_(0x5A)
    usk.build(pl, [to_dev(W) for W in Ws], sk)
    usk.check(pl)
    osk = orc.build_model(opl, Ws)
    np.testing.assert_array_equal(sk.cpu().numpy().view(np.uint16)[:opl.total_cells], osk)
    for l, (o, i) in enumerate(shapes):
        w = torch.empty(o, i, dtype=torch.bfloat16, device="cuda")
        usk.reconstruct(pl, sk, l, w)
        np.testing.assert_array_equal(w.cpu().view(torch.int16).numpy().view(np.uint16).reshape(-1),
                                      orc.reconstruct_rows(opl, osk, l).reshape(-1))


def test_xg_importance_classes_build(orc, usk):
    """USK-XG with C = 4 saliency classes scored per key group (ledger L33): the unit-major plan's bytes
    equal the oracle's, every key group is uniform, and the same plan in the query layout builds."""
    shapes = [(256, 512), (128, 256)]
    sal = [synth.saliency_like(i, 70 + k) for k, (o, i) in enumerate(shapes)]
    Ws = [synth.weights_bf16(o, i, 80 + k) for k, (o, i) in enumerate(shapes)]
    pl = usk.plan_allocation(shapes, bpw=0.5, hash="xg", seed=8, saliency=[torch.from_numpy(s).cuda() for s in sal])
    opl = orc.plan(shapes, 0.5, M=3, dtype=orc.BF16, hash_kind=orc.HASH_XG, seed=8, saliency=sal, C=4)
    sk = pl.new_sketch()
    usk.build(pl, [to_dev(W) for W in Ws], sk)
    osk = orc.build_model(opl, Ws)
    np.testing.assert_array_equal(sk.cpu().numpy().view(np.uint16)[:opl.total_cells], osk)
    for l in range(len(shapes)):
        cls, ncols = pl.export(l)[0], pl.export(l)[1]
        u0, u1 = opl.layer_units(l)
        np.testing.assert_array_equal(cls, opl.cls[u0:u1])
        np.testing.assert_array_equal(ncols, opl.ncols[u0:u1])
        assert (ncols.reshape(-1, 8) == ncols.reshape(-1, 8)[:, :1]).all()
    assert len(set(opl.ncols.tolist())) > 1  # the classes really differ


@pytest.mark.parametrize("layout", ["unit_major", "query"])
@pytest.mark.parametrize("crows", [None, (3, 3, 2, 2), (4, 3, 2, 1)])
def test_xg_importance_classes(orc, usk, crows, layout):
    """Importance classes (C = 4, optionally per-class rows, ledger L30) under USK-XG keys scored per
    key group (L33): groups uniform, so the grouped-key build runs; in the query layout the key groups
    are in class order with chunks cut at class boundaries (L34; no padding).  Bytes equal the
    oracle's (query bytes unpacked with tests/qlayout.py, from usk.h), reconstruction bit-exact, GEMV
    within 1e-5; a grouped call equals the single call bit for bit."""
    shapes = [(512, 1024), (300, 2048), (960, 256)]
    sal = [synth.saliency_like(i, 90 + k) for k, (o, i) in enumerate(shapes)]
    Ws = [synth.weights_bf16(o, i, 95 + k) for k, (o, i) in enumerate(shapes)]
    M = 3 if crows is None else max(crows)
    pl = usk.plan_allocation(shapes, bpw=0.5, rows=M, hash="xg", seed=9, n_classes=4, class_rows=crows,
                             saliency=[torch.from_numpy(s).cuda() for s in sal], layout=layout)
    opl = orc.plan(shapes, 0.5, M=M, dtype=orc.BF16, hash_kind=orc.HASH_XG, seed=9, saliency=sal, C=4,
                   class_rows=crows)
    sk = pl.new_sketch()
    sk.fill_(0xCD)
    usk.build(pl, [to_dev(W) for W in Ws], sk)
    usk.check(pl)
    osk = orc.build_model(opl, Ws)
    assert len(set(opl.ncols.tolist())) > 1
    if layout == "unit_major":
        np.testing.assert_array_equal(sk.cpu().numpy().view(np.uint16)[:opl.total_cells], osk)
    else:
        q = sk.cpu().numpy().view(np.uint16)
        for l in range(len(shapes)):
            u0, u1 = opl.layer_units(l)
            li = pl.layers[l]
            qb = q[li.qbyte_begin // 2:(li.qbyte_begin + li.qbytes) // 2]
            assert li.qbytes == sum(qlayout.layer_geometry(opl.ncols[u0:u1], M, opl.nrows[u0:u1], opl.cls[u0:u1])[1])
            cells, pad_ok = qlayout.unpack_layer(qb, opl.offsets[u0:u1 + 1], opl.ncols[u0:u1], opl.nrows[u0:u1], M,
                                                 opl.cls[u0:u1])
            np.testing.assert_array_equal(cells, osk[opl.offsets[u0]:opl.offsets[u1]])
            assert pad_ok
    for l, (o, i) in enumerate(shapes):
        ref = orc.reconstruct_rows(opl, osk, l)
        w = torch.empty(o, i, dtype=torch.bfloat16, device="cuda")
        usk.reconstruct(pl, sk, l, w)
        np.testing.assert_array_equal(w.cpu().view(torch.int16).numpy().view(np.uint16), ref)
        xb = synth.f32_to_bf16_bits(synth.vector(i, seed=200 + l)[0])
        xf = synth.bf16_bits_to_f32(xb).astype(np.float64)
        y = torch.empty((1, o), dtype=torch.float32, device="cuda")
        usk.linear(pl, sk, l, to_dev(xb).view(1, -1), y, usk.new_workspace(pl, l))
        y64 = orc.linear_rows(opl, osk, l, xf)[0]
        Wr = orc.value_of(ref, orc.BF16).reshape(o, i)
        assert gemv_err(y.cpu().numpy()[0], y64, xf, Wr) <= 1e-5
    xb = synth.f32_to_bf16_bits(synth.vector(2048, seed=300)[0])
    ys = [torch.empty(300, dtype=torch.float32, device="cuda") for _ in range(2)]
    usk.linear_batch(pl, sk, [1, 1], to_dev(xb), ys, usk.new_batch_workspace(pl, [1, 1]))
    y1 = torch.empty((1, 300), dtype=torch.float32, device="cuda")
    usk.linear(pl, sk, 1, to_dev(xb).view(1, -1), y1, usk.new_workspace(pl, 1))
    assert torch.equal(ys[0], y1[0]) and torch.equal(ys[1], y1[0])


def test_query_class_order_wide_chunks(orc, usk):
    """A class-ordered layer whose top class needs 64-unit chunks (a 128-unit chunk of its units would
    exceed shared memory) beside 256-unit chunks of the other classes: bytes, K3p reconstruction (one
    launch per width) and the K4p GEMV (one compute launch per width + one reduce) against the
    oracle, bf16 and fp32 x; an output shard equals the full call bit for bit."""
    shapes = [(2048, 512), (700, 512)]
    lv = np.array([1.0, 1.0, 40.0, 1.0], np.float32)
    rng = np.random.default_rng(3)
    sal = [np.repeat(lv, i // 4)[rng.permutation(i)].astype(np.float32) for (o, i) in shapes]
    Ws = [synth.weights_bf16(o, i, 61 + k) for k, (o, i) in enumerate(shapes)]
    pl = usk.plan_allocation(shapes, bpw=5.0, rows=3, hash="xg", layout="query", seed=12, n_classes=4,
                             saliency=[torch.from_numpy(s).cuda() for s in sal])
    opl = orc.plan(shapes, 5.0, M=3, dtype=orc.BF16, hash_kind=orc.HASH_XG, seed=12, saliency=sal, C=4)
    u0, u1 = opl.layer_units(0)
    ch, order = qlayout.chunks(opl.ncols[u0:u1], opl.nrows[u0:u1], 3, opl.cls[u0:u1])
    assert {c[2] for c in ch} >= {64, 256} and pl.layers[0].qchunk_units == 0, ch
    sk = pl.new_sketch()
    sk.fill_(0xCD)
    usk.build(pl, [to_dev(W) for W in Ws], sk)
    usk.check(pl)
    osk = orc.build_model(opl, Ws)
    q = sk.cpu().numpy().view(np.uint16)
    for l, (o, i) in enumerate(shapes):
        u0, u1 = opl.layer_units(l)
        li = pl.layers[l]
        qb = q[li.qbyte_begin // 2:(li.qbyte_begin + li.qbytes) // 2]
        cells, pad_ok = qlayout.unpack_layer(qb, opl.offsets[u0:u1 + 1], opl.ncols[u0:u1], opl.nrows[u0:u1], 3,
                                             opl.cls[u0:u1])
        np.testing.assert_array_equal(cells, osk[opl.offsets[u0]:opl.offsets[u1]])
        assert pad_ok
        ref = orc.reconstruct_rows(opl, osk, l)
        w = torch.empty(o, i, dtype=torch.bfloat16, device="cuda")
        usk.reconstruct(pl, sk, l, w)
        np.testing.assert_array_equal(w.cpu().view(torch.int16).numpy().view(np.uint16), ref)
    for xdt in (torch.bfloat16, torch.float32):
        xb = synth.f32_to_bf16_bits(synth.vector(512, seed=77)[0])
        x = to_dev(xb) if xdt == torch.bfloat16 else torch.from_numpy(synth.bf16_bits_to_f32(xb)).cuda()
        xf = synth.bf16_bits_to_f32(xb).astype(np.float64)
        ys = [torch.empty(o, dtype=torch.float32, device="cuda") for (o, i) in shapes]
        usk.linear_batch(pl, sk, [0, 1], x, ys, usk.new_batch_workspace(pl, [0, 1]))
        for l, (o, i) in enumerate(shapes):
            y64 = orc.linear_rows(opl, osk, l, xf)[0]
            Wr = orc.value_of(orc.reconstruct_rows(opl, osk, l), orc.BF16).reshape(o, i)
            assert gemv_err(ys[l].cpu().numpy(), y64, xf, Wr) <= 1e-5
        part = torch.empty(2048 - 333, dtype=torch.float32, device="cuda")
        usk.linear_batch(pl, sk, [0], x, [part], usk.new_batch_workspace(pl, [0], [(333, 2048)]), ranges=[(333, 2048)])
        assert torch.equal(part, ys[0][333:])


def test_query_importance_classes_chunk_aligned(orc, usk):
    """Importance classes whose units form whole chunks (saliency constant over runs of 256 input
    dims): the query layout holds them without padding, bit-exact against the oracle, and the
    grouped GEMV / reconstruction run on the packed kernels."""
    shapes = [(640, 1024), (200, 1024)]
    lv = np.array([1.0, 9.0, 3.0, 0.5], np.float32)
    sal = [np.repeat(lv, i // 4).astype(np.float32) for (o, i) in shapes]
    Ws = [synth.weights_bf16(o, i, 97 + k) for k, (o, i) in enumerate(shapes)]
    pl = usk.plan_allocation(shapes, bpw=0.5, rows=3, hash="xg", layout="query", seed=4, n_classes=4,
                             saliency=[torch.from_numpy(s).cuda() for s in sal])
    opl = orc.plan(shapes, 0.5, M=3, dtype=orc.BF16, hash_kind=orc.HASH_XG, seed=4, saliency=sal, C=4)
    assert len(set(opl.ncols.tolist())) >= 3
    sk = pl.new_sketch()
    sk.fill_(0xCD)
    usk.build(pl, [to_dev(W) for W in Ws], sk)
    usk.check(pl)
    osk = orc.build_model(opl, Ws)
    q = sk.cpu().numpy().view(np.uint16)
    assert sum(pl.layers[l].qbytes for l in range(len(shapes))) == 2 * opl.total_cells
    for l, (o, i) in enumerate(shapes):
        u0, u1 = opl.layer_units(l)
        li = pl.layers[l]
        qb = q[li.qbyte_begin // 2:(li.qbyte_begin + li.qbytes) // 2]
        cells, pad_ok = qlayout.unpack_layer(qb, opl.offsets[u0:u1 + 1], opl.ncols[u0:u1], opl.nrows[u0:u1], 3,
                                             opl.cls[u0:u1])
        np.testing.assert_array_equal(cells, osk[opl.offsets[u0]:opl.offsets[u1]])
        assert pad_ok
        ref = orc.reconstruct_rows(opl, osk, l)
        w = torch.empty(o, i, dtype=torch.bfloat16, device="cuda")
        usk.reconstruct(pl, sk, l, w)
        np.testing.assert_array_equal(w.cpu().view(torch.int16).numpy().view(np.uint16), ref)
    x = torch.from_numpy(synth.f32_to_bf16_bits(synth.vector(1024, seed=31)[0]).view(np.int16).copy()).view(torch.bfloat16).cuda()
    ys = [torch.empty(o, dtype=torch.float32, device="cuda") for (o, i) in shapes]
    usk.linear_batch(pl, sk, [0, 1], x, ys, usk.new_batch_workspace(pl, [0, 1]))
    xf = synth.bf16_bits_to_f32(x.cpu().view(torch.int16).numpy().view(np.uint16)).astype(np.float64)
    for l, (o, i) in enumerate(shapes):
        y64 = orc.linear_rows(opl, osk, l, xf)[0]
        Wr = orc.value_of(orc.reconstruct_rows(opl, osk, l), orc.BF16).reshape(o, i)
        assert gemv_err(ys[l].cpu().numpy(), y64, xf, Wr) <= 1e-5


def test_peer_allgather_epilogue_two_virtual_ranks(orc, usk):
    """usk_linear_batch_peers + usk_peer_wait (fused y all-gather) with two ranks simulated
    in one process on one GPU: each 'rank' computes its output shard and stores it into BOTH full-y
    buffers and both signal arrays; the waits then pass and both full y equal the single-GPU call bit
    for bit, over two epochs (graph-style replays).  No rank waits on a kernel of another (the launches
    are stream-ordered), so this checks the data placement and the flag protocol, not NVLink timing."""
    shapes = [(3000, 512), (700, 512), (1100, 512)]
    pl, opl, sk, osk, Ws = build_both(orc, usk, shapes)
    layers = [0, 1, 2]
    P = 2
    yfull = [[torch.zeros(o, dtype=torch.float32, device="cuda") for (o, i) in shapes] for _ in range(P)]
    sig = [torch.zeros(P, dtype=torch.int32, device="cuda") for _ in range(P)]
    epoch = [torch.zeros(1, dtype=torch.int32, device="cuda") for _ in range(P)]
    ref = [torch.empty(o, dtype=torch.float32, device="cuda") for (o, i) in shapes]
    for it in range(2):
        xb = synth.f32_to_bf16_bits(synth.vector(512, seed=40 + it)[0])
        x = torch.from_numpy(xb.view(np.int16).copy()).view(torch.bfloat16).cuda()
        usk.linear_batch(pl, sk, layers, x, ref, usk.new_batch_workspace(pl, layers))
        peers = []
        for r in range(P):
            ranges = [((o * r) // P, (o * (r + 1)) // P) for (o, i) in shapes]
            pr = usk.Peers(P, r, [[t.data_ptr() for t in yfull[q]] for q in range(P)], [s.data_ptr() for s in sig],
                           epoch[r])
            peers.append(pr)
            usk.linear_batch_peers(pl, sk, layers, x, pr, usk.new_batch_workspace(pl, layers, ranges), ranges=ranges)
        for r in range(P):
            usk.peer_wait(pl, peers[r])
        usk.check(pl)
        for r in range(P):
            assert int(epoch[r].item()) == it + 1
            assert sig[r].cpu().tolist() == [it + 1] * P
            for k in range(3):
                assert torch.equal(yfull[r][k], ref[k]), (it, r, k)


def test_query_reconstruct_batch(orc, usk):
    """usk_reconstruct_batch: consecutive layers with one in_features share a K3p launch; every layer's
    W' equals its single usk_reconstruct and the oracle, with padded leading dimensions."""
    shapes = [(2048, 512), (512, 512), (8192, 256), (130, 264), (96, 264)]
    pl, opl, sk, osk, Ws = build_both(orc, usk, shapes)
    outs = [torch.zeros(o, i + 8 * (k % 2), dtype=torch.bfloat16, device="cuda") for k, (o, i) in enumerate(shapes)]
    usk.reconstruct_batch(pl, sk, list(range(len(shapes))), outs)
    for l, (o, i) in enumerate(shapes):
        got = outs[l][:, :i].cpu().view(torch.int16).numpy().view(np.uint16)
        np.testing.assert_array_equal(got.reshape(-1), orc.reconstruct_rows(opl, osk, l).reshape(-1))


@pytest.mark.parametrize("M", [1, 2, 4])
def test_query_rows_1_2_4(orc, usk, M):
    """Query-layout kernels for M = 1, 2 and 4 sketch rows (template variants of K4p / K3p / the
    query write-out): bytes, reconstruction and GEMV against the oracle."""
    shapes = [(512, 512), (200, 264)]
    pl, opl, sk, osk, Ws = build_both(orc, usk, shapes, bpw=1.0, M=M)
    q = sk.cpu().numpy().view(np.uint16)
    for l, (o, i) in enumerate(shapes):
        u0, u1 = opl.layer_units(l)
        li = pl.layers[l]
        cells, pad_ok = qlayout.unpack_layer(q[li.qbyte_begin // 2:(li.qbyte_begin + li.qbytes) // 2],
                                             opl.offsets[u0:u1 + 1], opl.ncols[u0:u1], opl.nrows[u0:u1], M)
        np.testing.assert_array_equal(cells, osk[opl.offsets[u0]:opl.offsets[u1]])
        assert pad_ok
        w = torch.empty(o, i, dtype=torch.bfloat16, device="cuda")
        usk.reconstruct(pl, sk, l, w)
        np.testing.assert_array_equal(w.cpu().view(torch.int16).numpy().view(np.uint16).reshape(-1),
                                      orc.reconstruct_rows(opl, osk, l).reshape(-1))
        xb = synth.f32_to_bf16_bits(synth.vector(i, seed=l + 5)[0])
        xd = torch.from_numpy(xb.view(np.int16).copy()).view(torch.bfloat16).cuda()
        x64 = synth.bf16_bits_to_f32(xb).astype(np.float64)
        y = torch.empty(o, dtype=torch.float32, device="cuda")
        usk.linear(pl, sk, l, xd.view(1, -1), y.view(1, -1), usk.new_workspace(pl, l))
        Wr = orc.value_of(orc.reconstruct_rows(opl, osk, l), orc.BF16).reshape(o, i)
        assert gemv_err(y.cpu().numpy().astype(np.float64), orc.linear_rows(opl, osk, l, x64)[0], x64, Wr) <= 1e-5


def test_query_class_order_prefill(orc, usk):
    """T > 1 on a class-ordered plan (ledger L34): the batched reconstruction reads the chunk tables,
    then the tcgen05 GEMM; fp32 y within 1e-5 of the oracle's fp64 sums for every row of a few
    tokens, and the whole of y equal to the single-layer calls."""
    shapes = [(512, 1024), (300, 1024)]
    sal = [synth.saliency_like(i, 140 + k) for k, (o, i) in enumerate(shapes)]
    Ws = [synth.weights_bf16(o, i, 150 + k) for k, (o, i) in enumerate(shapes)]
    pl = usk.plan_allocation(shapes, bpw=0.5, rows=3, hash="xg", layout="query", seed=21, n_classes=4,
                             saliency=[torch.from_numpy(s).cuda() for s in sal], class_rows=(3, 3, 2, 2))
    opl = orc.plan(shapes, 0.5, M=3, dtype=orc.BF16, hash_kind=orc.HASH_XG, seed=21, saliency=sal, C=4,
                   class_rows=(3, 3, 2, 2))
    sk = pl.new_sketch()
    usk.build(pl, [to_dev(W) for W in Ws], sk)
    osk = orc.build_model(opl, Ws)
    T = 45
    xb = synth.f32_to_bf16_bits(synth.vector(1024, seed=8, T=T))
    x = to_dev(xb)
    ys = [torch.empty((T, o), dtype=torch.float32, device="cuda") for o, _ in shapes]
    usk.linear_batch_tokens(pl, sk, [0, 1], x, ys,
                            torch.zeros(usk.linear_batch_tokens_workspace_bytes(pl, [0, 1], T), dtype=torch.uint8,
                                        device="cuda"))
    x64 = synth.bf16_bits_to_f32(xb).astype(np.float64)
    for l, (o, i) in enumerate(shapes):
        ref = torch.empty((T, o), dtype=torch.float32, device="cuda")
        usk.linear(pl, sk, l, x, ref, usk.new_workspace(pl, l, T))
        assert torch.equal(ys[l], ref)
        y64 = orc.linear_rows(opl, osk, l, x64[:5])
        Wr = orc.value_of(orc.reconstruct_rows(opl, osk, l), orc.BF16).reshape(o, i)
        err = np.max(np.abs(ys[l].cpu().numpy()[:5] - y64) / np.maximum(np.abs(x64[:5]) @ np.abs(Wr).T, 1e-30))
        assert err <= 1e-5, err
