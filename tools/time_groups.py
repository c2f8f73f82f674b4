"""Per grouped call timing (tuning aid): Llama-3.2-1B block 0, q|k|v, o, gate|up, down as bench.py
groups them, each call timed alone with CUDA events behind an L2 flush, for each granularity.

  python tools/time_groups.py [--gran row outrow] [--reps 20]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2506_17255_b200 import usk  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--gran", nargs="+", default=["row", "outrow"])
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--bpw", type=float, default=0.5)
args = ap.parse_args()
dev = torch.device("cuda", 0)
shapes = synth.llama_block(2048, 512, 8192)
ws = [synth.torch_weights_bf16(o, i, synth.seed_for(3, 0, k), dev) for k, (o, i) in enumerate(shapes)]
groups = [[0, 1, 2], [3], [4, 5], [6]]
names = ["qkv", "o", "gate_up", "down"]
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for gran in args.gran:
    pl = usk.plan_allocation(shapes, bpw=args.bpw, rows=3, seed=0x5EED000000000003, granularity=gran)
    sk = pl.new_sketch(dev)
    usk.build(pl, ws, sk)
    usk.check(pl)
    row = []
    for g, nm in zip(groups, names):
        x = synth.torch_vector(shapes[g[0]][1], 7, dev, torch.bfloat16)[0]
        ys = [torch.empty(shapes[l][0], dtype=torch.float32, device=dev) for l in g]
        wsp = usk.new_batch_workspace(pl, g, device=dev)
        t = []
        for k in range(args.reps + 3):
            flush.fill_(k & 0xFF)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            usk.linear_batch(pl, sk, g, x, ys, wsp)
            b.record()
            b.synchronize()
            if k >= 3:
                t.append(a.elapsed_time(b) * 1000)
        w = sum(shapes[l][0] * shapes[l][1] for l in g)
        us = float(np.median(t))
        row.append(f"{nm} {us:7.2f} us ({w / us / 1e6:6.3f} Tw/s)")
    print(f"{gran:7s}: " + " | ".join(row), flush=True)
