"""Small end-to-end exercise of every kernel family for compute-sanitizer (SURVEY §5 / §4 tier 5;
tuning/evidence aid, not product):

  compute-sanitizer --tool {memcheck|racecheck|synccheck} python tools/sanitize_run.py

C1 (256x256 fp32, M=2, 1.0 bpw; ROW and LAYER units) and a scaled-down C2 MLP block (bf16,
M=3, 0.5 bpw, C=4 saliency classes): the plan kernels, the fast and generic builds (shared-memory
ring + red.shared.min, TMA tensor copies, mbarriers), reconstruct, the PDL-chained decode pair
(k_gemv_fast + k_gemv_reduce; two calls on one workspace, then a grouped call), Top-K, q4 states,
output-row units, and the prefill (reconstruct + the CTA-pair tcgen05 GEMM).  Results are checked
against the oracle on the small case so a sanitizer-induced change would also show."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402  (test infrastructure: the checker)
import synth  # noqa: E402
from paper_2506_17255_b200 import usk  # noqa: E402


def dev_bits(bits, dtype):
    if dtype == "bf16":
        return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16).copy()).view(torch.bfloat16).cuda()
    return torch.from_numpy(np.ascontiguousarray(bits)).cuda()


def c1():
    W = synth.weights_f32(256, 256, 1)
    for gran in ("row", "layer"):
        pl = usk.plan_allocation([(256, 256)], bpw=1.0, rows=2, granularity=gran, dtype="f32", seed=0x5EED000000000001)
        sk = pl.new_sketch()
        usk.build(pl, [dev_bits(W, "f32")], sk)
        usk.check(pl)
        Wr = torch.empty((256, 256), dtype=torch.float32, device="cuda")
        usk.reconstruct(pl, sk, 0, Wr)
        opl = oracle.plan([(256, 256)], 1.0, M=2, dtype=oracle.F32, gran=0 if gran == "row" else 1,
                          seed=0x5EED000000000001)
        osk = oracle.build_model(opl, [W])
        assert np.array_equal(Wr.cpu().numpy().view(np.uint32), oracle.reconstruct_rows(opl, osk, 0)), gran
        x = torch.from_numpy(synth.vector(256, seed=2)[0]).cuda()
        y = torch.empty((1, 256), dtype=torch.float32, device="cuda")
        usk.linear(pl, sk, 0, x.view(1, -1), y, usk.new_workspace(pl, 0))
    print("c1 ok")


def c2_small():
    shapes = [(2048, 512), (2048, 512), (512, 2048)]
    Ws = [synth.weights_bf16(o, i, 30 + k) for k, (o, i) in enumerate(shapes)]
    sal = [torch.from_numpy(synth.saliency_like(i, 40 + k)).cuda() for k, (o, i) in enumerate(shapes)]
    pl = usk.plan_allocation(shapes, bpw=0.5, rows=3, n_classes=4, seed=7, saliency=sal)
    sk = pl.new_sketch()
    dW = [dev_bits(W, "bf16") for W in Ws]
    usk.build(pl, dW, sk)
    usk.check(pl)
    for l, (o, i) in enumerate(shapes):
        Wr = torch.empty((o, i), dtype=torch.bfloat16, device="cuda")
        usk.reconstruct(pl, sk, l, Wr)
    # decode: two calls on one workspace (the "left zeroed" contract), then the grouped call
    xb = synth.f32_to_bf16_bits(synth.vector(512, seed=5)[0])
    x = dev_bits(xb, "bf16")
    ws = usk.new_workspace(pl, 0)
    y1 = torch.empty((1, 2048), dtype=torch.float32, device="cuda")
    y2 = torch.empty_like(y1)
    usk.linear(pl, sk, 0, x.view(1, -1), y1, ws)
    usk.linear(pl, sk, 0, x.view(1, -1), y2, ws)
    assert torch.equal(y1, y2)
    ys = [torch.empty(2048, dtype=torch.float32, device="cuda") for _ in range(2)]
    usk.linear_batch(pl, sk, [0, 1], x, ys, usk.new_batch_workspace(pl, [0, 1]))
    assert torch.equal(ys[0], y1[0])
    xd = dev_bits(synth.f32_to_bf16_bits(synth.vector(2048, seed=6)[0]), "bf16")
    yd = torch.empty((1, 512), dtype=torch.float32, device="cuda")
    usk.linear(pl, sk, 2, xd.view(1, -1), yd, usk.new_workspace(pl, 2))
    # prefill: K3 into the workspace + the CTA-pair tcgen05 GEMM
    T = 256
    X = synth.torch_vector(512, 8, "cuda", torch.bfloat16, T=T)
    Y = torch.empty((T, 2048), dtype=torch.bfloat16, device="cuda")
    usk.linear(pl, sk, 0, X, Y, usk.new_workspace(pl, 0, T))
    torch.cuda.synchronize()
    print("c2-small ok")


def extras():
    shapes = [(512, 256)]
    W = synth.weights_bf16(512, 256, 9)
    for kw in (dict(topk=64, bpw=8.0), dict(state_bits=4, group_size=128, bpw=1.0), dict(granularity="outrow", bpw=1.0)):
        pl = usk.plan_allocation(shapes, rows=3, seed=3, **kw)
        sk = pl.new_sketch()
        usk.build(pl, [dev_bits(W, "bf16")], sk)
        usk.check(pl)
        Wr = torch.empty((512, 256), dtype=torch.bfloat16, device="cuda")
        usk.reconstruct(pl, sk, 0, Wr)
        x = torch.from_numpy(synth.vector(256, seed=1)[0]).cuda()
        y = torch.empty((1, 512), dtype=torch.float32, device="cuda")
        usk.linear(pl, sk, 0, x.view(1, -1), y, usk.new_workspace(pl, 0))
        assert torch.isfinite(y).all()
    torch.cuda.synchronize()
    print("extras ok")


if __name__ == "__main__":
    torch.cuda.set_device(0)
    c1()
    c2_small()
    extras()
    print("sanitize_run done")
