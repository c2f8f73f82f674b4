"""Config-4 prefill pass timing variants (tuning aid): all 112 Llama-3.2-1B linears at T = 16384 in model
order through usk_linear (K3p reconstruct into the workspace + the tcgen05 GEMM), the same grouped as
q|k|v, o, gate|up, down through usk_linear_batch_tokens (one reconstruction + one GEMM per group), eager
vs captured in one CUDA graph, plus the 112 reconstructions alone: where the pass time goes.
  python tools/prefill_pass.py [--bpw 0.5] [--reps 5]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2506_17255_b200 import usk  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--bpw", type=float, default=0.5)
ap.add_argument("--reps", type=int, default=5)
args = ap.parse_args()
dev = torch.device("cuda", 0)
shapes = synth.llama32_1b_shapes()
pl = usk.plan_allocation(shapes, bpw=args.bpw, rows=3, seed=0x5EED000000000003, hash="xg", layout="query")
sk = pl.new_sketch(dev)
usk.build(pl, [synth.torch_weights_bf16(o, i, synth.seed_for(3, l // 7, l % 7), dev) for l, (o, i) in enumerate(shapes)], sk)
T = 16384
Xp = synth.torch_vector(8192, 77, dev, torch.bfloat16, T=T).reshape(-1)
Yp = torch.empty(T * 8192, dtype=torch.bfloat16, device=dev)
Xw = {i: Xp[:T * i].view(T, i) for i in {i for _, i in shapes}}
Yw = {o: Yp[:T * o].view(T, o) for o in {o for o, _ in shapes}}
Yp2 = torch.empty(T * 16384, dtype=torch.bfloat16, device=dev)
wsp = torch.zeros(max(usk.linear_workspace_bytes(pl, l, T) for l in range(len(shapes))) * 2, dtype=torch.uint8, device=dev)
st = torch.cuda.Stream(device=dev)


def pass_full():
    for l, (o, i) in enumerate(shapes):
        usk.linear(pl, sk, l, Xw[i], Yw[o], wsp, stream=st)


groups = []
for b in range(len(shapes) // 7):
    groups += [[7 * b, 7 * b + 1, 7 * b + 2], [7 * b + 3], [7 * b + 4, 7 * b + 5], [7 * b + 6]]
Yg = []
for g in groups:
    ys, off = [], 0
    for l in g:
        ys.append(Yp2[off:off + T * shapes[l][0]].view(T, shapes[l][0]))
        off += T * shapes[l][0]
    Yg.append(ys)


def pass_grouped():
    for gi, g in enumerate(groups):
        usk.linear_batch_tokens(pl, sk, g, Xw[shapes[g[0]][1]], Yg[gi], wsp, stream=st)


# pipelined: the next group's W' rebuilt (usk_reconstruct_batch) on a side stream into the other of
# two workspaces while this group's GEMM (usk_gemm_tokens) runs
side = torch.cuda.Stream(device=dev)
gmax = max(sum(shapes[l][0] for l in g) * shapes[g[0]][1] for g in groups)
wsx = [torch.empty(gmax, dtype=torch.bfloat16, device=dev) for _ in range(2)]


def w_views(gi):
    g = groups[gi]
    i = shapes[g[0]][1]
    out, off = [], 0
    for l in g:
        o = shapes[l][0]
        out.append(wsx[gi % 2][off:off + o * i].view(o, i))
        off += o * i
    return out


def pass_pipelined():
    n = len(groups)
    ev_r = [torch.cuda.Event() for _ in range(n)]
    ev_g = [torch.cuda.Event() for _ in range(n)]
    start = torch.cuda.Event()
    start.record(st)
    side.wait_event(start)
    with torch.cuda.stream(side):
        usk.reconstruct_batch(pl, sk, groups[0], w_views(0), stream=side)
        ev_r[0].record(side)
    for gi, g in enumerate(groups):
        if gi + 1 < n:
            if gi >= 1:
                side.wait_event(ev_g[gi - 1])  # its workspace is free once GEMM gi-1 is done
            with torch.cuda.stream(side):
                usk.reconstruct_batch(pl, sk, groups[gi + 1], w_views(gi + 1), stream=side)
                ev_r[gi + 1].record(side)
        st.wait_event(ev_r[gi])
        i = shapes[g[0]][1]
        usk.gemm_tokens(Xw[i], wsx[gi % 2][:sum(shapes[l][0] for l in g) * i].view(-1, i),
                        [shapes[l][0] for l in g], Yg[gi], stream=st)
        ev_g[gi].record(st)
    st.wait_stream(side)


def pass_recon():
    for l, (o, i) in enumerate(shapes):
        usk.reconstruct(pl, sk, l, wsp[:o * i * 2].view(torch.bfloat16).view(o, i), stream=st)


def timed(fn, graph):
    with torch.cuda.stream(st):
        fn()
    torch.cuda.synchronize()
    g = None
    if graph:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            fn()
    ts = []
    for _ in range(args.reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(st):
            a.record(st)
            g.replay() if g is not None else fn()
            b.record(st)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


out = {"bpw": args.bpw}
for name, fn in (("pass", pass_full), ("pass_grouped", pass_grouped), ("pass_pipelined", pass_pipelined),
                 ("recon_only", pass_recon)):
    for graph in (False, True):
        out[f"{name}_{'graph' if graph else 'eager'}_ms"] = timed(fn, graph)
print(json.dumps(out), flush=True)
# the pipelined pass writes the same Y as the grouped one (same W', same GEMM)
with torch.cuda.stream(st):
    pass_grouped()
torch.cuda.synchronize()
ref = Yp2.clone()
Yp2.zero_()
with torch.cuda.stream(st):
    pass_pipelined()
torch.cuda.synchronize()
print(json.dumps({"pipelined_equals_grouped": bool(torch.equal(ref, Yp2))}), flush=True)
