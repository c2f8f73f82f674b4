"""Standalone reconstruct (K3) timing (tuning aid): usk_reconstruct of all 112 Llama-3.2-1B linears
into one scratch buffer, captured as one CUDA graph, L2 flushed before each replay (as bench.py's
reconstruct_standalone); plus one Llama-3.2-1B block's prefill (usk_linear T = 16384, 7 linears)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2506_17255_b200 import usk  # noqa: E402

dev = torch.device("cuda", 0)
shapes = synth.llama32_1b_shapes()
pl = usk.plan_allocation(shapes, bpw=0.5, rows=3, seed=0x5EED000000000003)
sk = pl.new_sketch(dev)
ws = [synth.torch_weights_bf16(o, i, synth.seed_for(3, l // 7, l % 7), dev) for l, (o, i) in enumerate(shapes)]
usk.build(pl, ws, sk)
del ws
stream = torch.cuda.Stream(device=dev)
scratch = torch.empty(max(o * i for o, i in shapes), dtype=torch.bfloat16, device=dev)


def rec_all():
    for l, (o, i) in enumerate(shapes):
        usk.reconstruct(pl, sk, l, scratch[:o * i].view(o, i), stream=stream)


with torch.cuda.stream(stream):
    rec_all()
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=stream):
    rec_all()
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
t = []
for k in range(7):
    with torch.cuda.stream(stream):
        flush.fill_(k)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        g.replay()
        b.record(stream)
    b.synchronize()
    t.append(a.elapsed_time(b))
ms = float(np.median(t))
n = sum(o * i for o, i in shapes)
# one block's prefill
T = 16384
X = synth.torch_vector(8192, 5, dev, torch.bfloat16, T=T).reshape(-1)
Y = torch.empty(T * 8192, dtype=torch.bfloat16, device=dev)
wsp = torch.zeros(max(usk.linear_workspace_bytes(pl, l, T) for l in range(7)), dtype=torch.uint8, device=dev)


def block():
    for l in range(7):
        o, i = shapes[l]
        usk.linear(pl, sk, l, X[:T * i].view(T, i), Y[:T * o].view(T, o), wsp, stream=stream)


with torch.cuda.stream(stream):
    block()
tb = []
for k in range(5):
    with torch.cuda.stream(stream):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        block()
        b.record(stream)
    b.synchronize()
    tb.append(a.elapsed_time(b))
print(json.dumps({"reconstruct_112_ms": ms, "weights_per_s": n / (ms * 1e-3), "GB_per_s_written": n * 2 / (ms * 1e-3) / 1e9,
                  "prefill_block_ms": float(np.median(tb))}))
