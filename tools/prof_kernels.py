"""Small driver for ncu: builds the Llama-3.2-1B block-0 sketch and launches the hot kernels
(build, reconstruct, sketch-GEMV) a few times each on cuda:0.

  python tools/prof_kernels.py [--layers q,gate,down] [--reps 3]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2506_17255_b200 import usk  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--bpw", type=float, default=0.5)
args = ap.parse_args()
dev = torch.device("cuda", 0)
shapes = synth.llama_block(2048, 512, 8192)
pl = usk.plan_allocation(shapes, bpw=args.bpw, rows=3, seed=0x5EED000000000003)
sk = pl.new_sketch(dev)
ws = [synth.torch_weights_bf16(o, i, synth.seed_for(3, 0, k), dev) for k, (o, i) in enumerate(shapes)]
for _ in range(args.reps):
    usk.build(pl, ws, sk)
usk.check(pl)
scratch = torch.empty(8192 * 2048, dtype=torch.bfloat16, device=dev)
for _ in range(args.reps):
    for l, (o, i) in enumerate(shapes):
        usk.reconstruct(pl, sk, l, scratch[:o * i].view(o, i))
for l, (o, i) in enumerate(shapes):
    x = synth.torch_vector(i, 1000 + l, dev, torch.bfloat16)
    y = torch.empty((1, o), dtype=torch.float32, device=dev)
    w = usk.new_workspace(pl, l, device=dev)
    for _ in range(args.reps):
        usk.linear(pl, sk, l, x, y, w)
torch.cuda.synchronize()
print("ok")
