"""GPU tests of the finetuning operators (Figure 4): the
fake-compress STE op (forward = build + reconstruct, bit-exact vs the oracle; backward = identity;
finite differences of a loss w.r.t. the decompressed weights) and the aggregated-gradient
baseline (bit-exact vs the oracle's 2^-48 fixed-point sums, ledger L26)."""
import numpy as np
import pytest

import synth
from test_gpu_parity import DT, to_dev, w_bits

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def usk():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2506_17255_b200 import usk as u
    return u


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_fake_compress_forward_backward(orc, usk, dtype):
    from paper_2506_17255_b200.ste import fake_compress
    shapes = [(96, 64), (128, 96)]
    pl = usk.plan_allocation(shapes, bpw=2.0, rows=3, dtype=dtype, seed=17)
    opl = orc.plan(shapes, 2.0, M=3, dtype=DT[dtype], seed=17)
    sk = pl.new_sketch()
    Ws = [synth.weights_bf16(o, i, 40 + l) if dtype == "bf16" else synth.weights_f32(o, i, 40 + l)
          for l, (o, i) in enumerate(shapes)]
    for l, W in enumerate(Ws):
        Wd = to_dev(W, dtype).requires_grad_(True)
        Wp = fake_compress(Wd, pl, l, sk)
        osk = orc.build_model(opl, Ws)
        np.testing.assert_array_equal(w_bits(Wp.detach(), dtype), orc.reconstruct_rows(opl, osk, l))
        G = torch.randn_like(Wp)
        Wp.backward(G)
        assert torch.equal(Wd.grad, G)  # straight-through: bit-identical


def test_fake_compress_rebuilds_every_call(orc, usk):
    # the bindings follow the current weights ("may vary during finetuning")
    from paper_2506_17255_b200.ste import fake_compress
    o, i = 64, 64
    pl = usk.plan_allocation([(o, i)], bpw=2.0, rows=3, dtype="f32", seed=5)
    opl = orc.plan([(o, i)], 2.0, M=3, dtype=orc.F32, seed=5)
    sk = pl.new_sketch()
    W = synth.weights_f32(o, i, 1)
    W2 = W.copy()
    W2[::3] *= -2.5
    for Wn in (W, W2):
        Wp = fake_compress(to_dev(Wn, "f32"), pl, 0, sk)
        np.testing.assert_array_equal(w_bits(Wp, "f32"), orc.reconstruct_rows(opl, orc.build_model(opl, [Wn]), 0))


def test_ste_finite_differences(usk):
    # SPEC ste_backward: composed with the fake-compress forward, the gradient matches central finite
    # differences of the loss w.r.t. the decompressed weights (10^-4 relative, 8x8 layer)
    from paper_2506_17255_b200.ste import fake_compress
    o, i = 8, 8
    pl = usk.plan_allocation([(o, i)], bpw=16.0, rows=3, dtype="f32", seed=2)
    sk = pl.new_sketch()
    g = torch.Generator().manual_seed(0)
    W = (torch.randn(o, i, generator=g, dtype=torch.float64) * 0.5).float().cuda().requires_grad_(True)
    X = torch.randn(16, i, generator=g, dtype=torch.float64).cuda()
    Y = torch.randn(16, o, generator=g, dtype=torch.float64).cuda()

    def loss_of(Wp):
        return ((X @ Wp.double().T - Y) ** 2).sum()

    Wp = fake_compress(W, pl, 0, sk)
    loss_of(Wp).backward()
    Wd = Wp.detach().double()
    h = 1e-4
    fd = torch.zeros_like(Wd)
    for a in range(o):
        for b in range(i):
            E = torch.zeros_like(Wd)
            E[a, b] = h
            fd[a, b] = (loss_of(Wd + E) - loss_of(Wd - E)) / (2 * h)
    rel = ((W.grad.double() - fd).abs() / fd.abs().clamp_min(1.0)).max().item()
    assert rel <= 1e-4, rel


@pytest.mark.parametrize("case", [
    ([(96, 64), (40, 96)], "row", 1, 3, "bf16", "bf16"),
    ([(300, 96)], "row", 1, 2, "f32", "f32"),
    ([(130, 64)], "row", 2, 3, "bf16", "f32"),
    ([(64, 32), (96, 64)], "layer", 1, 3, "bf16", "bf16"),
    ([(70, 64)], "row", 1, 1, "f32", "f32"),
], ids=lambda c: f"{c[1]}-g{c[2]}-M{c[3]}-{c[4]}-grad{c[5]}")
def test_aggregate_grad_bit_exact(orc, usk, case):
    shapes, gran, g, M, dtype, gdt = case
    pl = usk.plan_allocation(shapes, bpw=2.0, rows=M, granularity=gran, dims_per_unit=g, dtype=dtype, seed=31)
    opl = orc.plan(shapes, 2.0, M=M, dtype=DT[dtype], gran=1 if gran == "layer" else 0, g=g, seed=31)
    ws = None
    for l, (o, i) in enumerate(shapes):
        grad = synth.weights_f32(o, i, 70 + l) * 10.0
        if gdt == "bf16":
            gb = synth.f32_to_bf16_bits(grad)
            gd = torch.from_numpy(gb.view(np.int16).copy()).view(torch.bfloat16).cuda()
            gv = synth.bf16_bits_to_f32(gb).astype(np.float64)
        else:
            gd = torch.from_numpy(grad).cuda()
            gv = grad.astype(np.float64)
        n = pl.layers[l].n_cells
        out = torch.empty(n, dtype=torch.float32, device="cuda")
        if ws is None:
            ws = torch.zeros(max(pl.layers[k].n_cells for k in range(len(shapes))) * 8, dtype=torch.uint8,
                             device="cuda")
        usk.aggregate_grad(pl, l, gd, out, ws)
        want = orc.aggregate_grad(opl, l, gv)
        np.testing.assert_array_equal(out.cpu().numpy().view(np.uint32), want.view(np.uint32))
        assert int(ws.count_nonzero()) == 0  # workspace left zero-filled
