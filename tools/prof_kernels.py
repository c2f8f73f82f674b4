"""Small driver for ncu: builds the Llama-3.2-1B block-0 sketch and launches the hot kernels in
the order: grouped sketch-GEMVs (q|k|v, o, gate|up, down -- as bench.py launches them), the build,
the reconstruction of gate, and (with --prefill) one 2048-token prefill of gate|up (batched
reconstruction + one tcgen05 GEMM).  Default plan: USK-XG keys, query layout (the bench's).

  python tools/prof_kernels.py [--reps 1] [--prefill]
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
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--bpw", type=float, default=0.5)
ap.add_argument("--prefill", action="store_true")
ap.add_argument("--gran", default="row")
ap.add_argument("--layout", default="query", choices=["query", "unit_major"])
args = ap.parse_args()
dev = torch.device("cuda", 0)
shapes = synth.llama_block(2048, 512, 8192)
pl = usk.plan_allocation(shapes, bpw=args.bpw, rows=3, seed=0x5EED000000000003, granularity=args.gran,
                         **({"hash": "xg", "layout": "query"} if args.layout == "query" else {}))
sk = pl.new_sketch(dev)
ws = [synth.torch_weights_bf16(o, i, synth.seed_for(3, 0, k), dev) for k, (o, i) in enumerate(shapes)]
torch.cuda.synchronize()
# the build itself is launched below (after the GEMVs) for the capture order; build once first
# without profiling interest would add a kernel, so the GEMV inputs use a build done here
usk.build(pl, ws, sk)
usk.check(pl)
groups = [[0, 1, 2], [3], [4, 5], [6]]
for _ in range(args.reps):
    for g in groups:
        x = synth.torch_vector(shapes[g[0]][1], 7, dev, torch.bfloat16)[0]
        ys = [torch.empty(shapes[l][0], dtype=torch.float32, device=dev) for l in g]
        usk.linear_batch(pl, sk, g, x, ys, usk.new_batch_workspace(pl, g, device=dev))
for _ in range(args.reps):
    usk.build(pl, ws, sk)
scratch = torch.empty(8192 * 2048, dtype=torch.bfloat16, device=dev)
for _ in range(args.reps):
    usk.reconstruct(pl, sk, 4, scratch.view(8192, 2048))
if args.prefill:
    T = 2048
    X = synth.torch_vector(2048, 5, dev, torch.bfloat16, T=T)
    ys = [torch.empty((T, 8192), dtype=torch.bfloat16, device=dev) for _ in range(2)]
    wsp = torch.zeros(usk.linear_batch_tokens_workspace_bytes(pl, [4, 5], T), dtype=torch.uint8, device=dev)
    usk.linear_batch_tokens(pl, sk, [4, 5], X, ys, wsp)  # gate|up: one reconstruction + one GEMM
torch.cuda.synchronize()
print("ok")
