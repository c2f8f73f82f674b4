"""Prefill path (usk_linear with T > 1): reconstruct the output-row slice of W' into the workspace,
then the tcgen05 GEMM.  Tolerance (BASELINE.json north_star, L23): scaled error
max |Y - Y64| / sum_j |x_tj w'_oj| <= 2e-2 for bf16 Y, <= 1e-5 for fp32 Y (fp32 accumulation)."""
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


def _bf16_dev(bits):
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16).copy()).view(torch.bfloat16).cuda()


@pytest.mark.parametrize("shape,T", [((256, 128), 128), ((512, 256), 3), ((300, 192), 130), ((384, 640), 257),
                                     ((1000, 64), 1000)])
@pytest.mark.parametrize("ydt", ["bf16", "f32"])
def test_prefill_matches_oracle(orc, usk, shape, T, ydt):
    o, i = shape
    W = synth.weights_bf16(o, i, seed=o + i)
    pl = usk.plan_allocation([shape], bpw=1.0, rows=3, seed=77)
    opl = orc.plan([shape], 1.0, M=3, dtype=orc.BF16, seed=77)
    sk = pl.new_sketch()
    usk.build(pl, [_bf16_dev(W)], sk)
    osk = orc.build_model(opl, [W])
    xb = synth.f32_to_bf16_bits(synth.vector(i, seed=T, T=T))
    x = _bf16_dev(xb)
    y = torch.empty((T, o), dtype=torch.bfloat16 if ydt == "bf16" else torch.float32, device="cuda")
    usk.linear(pl, sk, 0, x, y, usk.new_workspace(pl, 0, T))
    x64 = synth.bf16_bits_to_f32(xb).astype(np.float64)
    rows = np.arange(0, o) if o * T <= 300_000 else np.random.default_rng(0).choice(o, 64, replace=False)
    y64 = np.stack([orc.linear_rows(opl, osk, 0, x64, r, r + 1)[:, 0] for r in rows], 1)
    Wr = orc.value_of(orc.reconstruct_rows(opl, osk, 0), orc.BF16).reshape(o, i)[rows]
    got = y.float().cpu().numpy().astype(np.float64)[:, rows]
    scale = np.abs(x64) @ np.abs(Wr).T
    err = np.max(np.abs(got - y64) / np.maximum(scale, 1e-30))
    assert err <= (2e-2 if ydt == "bf16" else 1e-5), err
    big = np.abs(y64) >= 1e-3 * np.sqrt(np.mean(y64 ** 2))
    rel = np.max(np.abs(got - y64)[big] / np.abs(y64)[big])
    assert rel <= (1e-2 if ydt == "bf16" else 1e-3), rel


def test_prefill_output_shard(orc, usk):
    o, i, T = 512, 256, 200
    W = synth.weights_bf16(o, i, seed=1)
    pl = usk.plan_allocation([(o, i)], bpw=1.0, rows=3, seed=3)
    sk = pl.new_sketch()
    usk.build(pl, [_bf16_dev(W)], sk)
    x = _bf16_dev(synth.f32_to_bf16_bits(synth.vector(i, seed=2, T=T)))
    full = torch.empty((T, o), dtype=torch.float32, device="cuda")
    usk.linear(pl, sk, 0, x, full, usk.new_workspace(pl, 0, T))
    part = torch.empty((T, o - 100), dtype=torch.float32, device="cuda")
    usk.linear(pl, sk, 0, x, part, usk.new_workspace(pl, 0, T, 100, o), out_begin=100, out_end=o)
    assert torch.equal(part, full[:, 100:])


def test_prefetch_l2_is_a_pure_hint(usk):
    """usk_prefetch_l2 changes no result (decode and prefill bit-equal with and without it) and
    rejects a layer range outside [0, n_layers)."""
    shapes = [(512, 256), (256, 512)]
    pl = usk.plan_allocation(shapes, bpw=0.5, rows=3, seed=5)
    sk = pl.new_sketch()
    usk.build(pl, [_bf16_dev(synth.weights_bf16(o, i, seed=o)) for o, i in shapes], sk)
    outs = []
    for pf in (False, True):
        if pf:
            usk.prefetch_l2(pl, sk)
            usk.prefetch_l2(pl, sk, 1, 2)
            usk.prefetch_l2(pl, sk, 1, 1)  # empty range: no launch
        ys = []
        for l, (o, i) in enumerate(shapes):
            for T in (1, 100):
                x = _bf16_dev(synth.f32_to_bf16_bits(synth.vector(i, seed=l, T=T)))
                y = torch.empty((T, o), dtype=torch.float32, device="cuda")
                usk.linear(pl, sk, l, x, y, usk.new_workspace(pl, l, T))
                ys.append(y)
        torch.cuda.synchronize()
        outs.append(ys)
    for a, b in zip(*outs):
        assert torch.equal(a, b)
    with pytest.raises(usk.UskError):
        usk.prefetch_l2(pl, sk, 0, 3)
    with pytest.raises(usk.UskError):
        usk.prefetch_l2(pl, sk, 2, 1)


def _group(orc, usk, shapes, layout, seed=21):
    Ws = [synth.weights_bf16(o, i, seed=seed + k) for k, (o, i) in enumerate(shapes)]
    kw = dict(hash="xg", layout="query") if layout == "query" else {}
    pl = usk.plan_allocation(shapes, bpw=1.0, rows=3, seed=seed, **kw)
    opl = orc.plan(shapes, 1.0, M=3, dtype=orc.BF16, seed=seed,
                   hash_kind=orc.HASH_XG if layout == "query" else orc.HASH_X)
    sk = pl.new_sketch()
    usk.build(pl, [_bf16_dev(W) for W in Ws], sk)
    return pl, opl, sk, orc.build_model(opl, Ws)


@pytest.mark.parametrize("layout", ["unit_major", "query"])
@pytest.mark.parametrize("shapes", [[(96, 256), (160, 256), (300, 256)],   # one GEMM, ragged last layer
                                    [(100, 256), (64, 256)]],               # 100 % 32 != 0: layer by layer
                         ids=["fused", "sequential"])
@pytest.mark.parametrize("T", [3, 130, 257])
def test_batch_tokens_matches_oracle_and_single_calls(orc, usk, layout, shapes, T):
    """usk_linear_batch_tokens (the group's W' rebuilt once, one GEMM with per-layer output
    segments): every y[k] equals usk_linear of layer k bit for bit (same products, same K order), and
    the fp32 results are within 1e-5 of the oracle's fp64 sums."""
    pl, opl, sk, osk = _group(orc, usk, shapes, layout)
    i = shapes[0][1]
    xb = synth.f32_to_bf16_bits(synth.vector(i, seed=T + 5, T=T))
    x = _bf16_dev(xb)
    x64 = synth.bf16_bits_to_f32(xb).astype(np.float64)
    layers = list(range(len(shapes)))
    for dt in (torch.float32, torch.bfloat16):
        ys = [torch.full((T, o), 7.0, dtype=dt, device="cuda") for (o, _) in shapes]
        ws = torch.zeros(usk.linear_batch_tokens_workspace_bytes(pl, layers, T), dtype=torch.uint8, device="cuda")
        usk.linear_batch_tokens(pl, sk, layers, x, ys, ws)
        for l, (o, _) in enumerate(shapes):
            ref = torch.empty((T, o), dtype=dt, device="cuda")
            usk.linear(pl, sk, l, x, ref, usk.new_workspace(pl, l, T))
            assert torch.equal(ys[l], ref), (l, dt)
            if dt == torch.float32:
                y64 = orc.linear_rows(opl, osk, l, x64)
                Wr = orc.value_of(orc.reconstruct_rows(opl, osk, l), orc.BF16).reshape(o, i)
                err = np.max(np.abs(ys[l].cpu().numpy() - y64) / np.maximum(np.abs(x64) @ np.abs(Wr).T, 1e-30))
                assert err <= 1e-5, err


def test_batch_tokens_ranges_and_rejections(orc, usk):
    """Output ranges (sharded prefill) run layer by layer with the same bytes as usk_linear on each
    range; fp32 x is refused with USK_EUNSUPPORTED."""
    shapes = [(256, 128), (192, 128)]
    pl, opl, sk, osk = _group(orc, usk, shapes, "query", seed=5)
    T = 77
    x = _bf16_dev(synth.f32_to_bf16_bits(synth.vector(128, seed=9, T=T)))
    ranges = [(32, 200), (0, 100)]
    ys = [torch.empty((T, b - a), dtype=torch.float32, device="cuda") for a, b in ranges]
    ws = torch.zeros(usk.linear_batch_tokens_workspace_bytes(pl, [0, 1], T, ranges), dtype=torch.uint8, device="cuda")
    usk.linear_batch_tokens(pl, sk, [0, 1], x, ys, ws, ranges=ranges)
    for l, (a, b) in enumerate(ranges):
        ref = torch.empty((T, b - a), dtype=torch.float32, device="cuda")
        usk.linear(pl, sk, l, x, ref, usk.new_workspace(pl, l, T, a, b), out_begin=a, out_end=b)
        assert torch.equal(ys[l], ref)
    with pytest.raises(usk.UskError) as e:
        usk.linear_batch_tokens(pl, sk, [0, 1], x.float(), [torch.empty((T, o), device="cuda") for o, _ in shapes], ws)
    assert e.value.status == usk.EUNSUPPORTED


def test_gemm_tokens_equals_batch_tokens(orc, usk):
    """usk_gemm_tokens (the computation stage alone, on W' rebuilt by usk_reconstruct_batch) gives the
    bytes of usk_linear_batch_tokens; rejects an inner block with rows % 32 != 0."""
    shapes = [(96, 256), (160, 256), (300, 256)]
    pl, opl, sk, osk = _group(orc, usk, shapes, "query", seed=33)
    T = 70
    x = _bf16_dev(synth.f32_to_bf16_bits(synth.vector(256, seed=4, T=T)))
    layers = [0, 1, 2]
    ref = [torch.empty((T, o), dtype=torch.float32, device="cuda") for o, _ in shapes]
    usk.linear_batch_tokens(pl, sk, layers, x, ref,
                            torch.zeros(usk.linear_batch_tokens_workspace_bytes(pl, layers, T), dtype=torch.uint8,
                                        device="cuda"))
    w = torch.empty((sum(o for o, _ in shapes), 256), dtype=torch.bfloat16, device="cuda")
    views, r = [], 0
    for o, _ in shapes:
        views.append(w[r:r + o])
        r += o
    usk.reconstruct_batch(pl, sk, layers, views)
    ys = [torch.empty((T, o), dtype=torch.float32, device="cuda") for o, _ in shapes]
    usk.gemm_tokens(x, w, [o for o, _ in shapes], ys)
    for a, b in zip(ys, ref):
        assert torch.equal(a, b)
    with pytest.raises(usk.UskError):
        usk.gemm_tokens(x, w[:100 + 160], [100, 160], [torch.empty((T, 100), device="cuda"),
                                                       torch.empty((T, 160), device="cuda")])
