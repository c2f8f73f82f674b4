"""Where the config-4 prefill time goes, per linear of a Llama-3.2-1B block at T = 16384:
usk.linear (K3 reconstruct into the workspace + the tcgen05 GEMM), usk.reconstruct alone, and
cuBLAS (torch.matmul) on the same X and a dense bf16 W' of the same shape, as the library GEMM
beside ours.  CUDA events on one stream, median of 5 after 2 warm-ups.

  python tools/prefill_split.py [--T 16384] [--bpw 0.5]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2506_17255_b200 import usk  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--T", type=int, default=16384)
ap.add_argument("--bpw", type=float, default=0.5)
args = ap.parse_args()
dev = torch.device("cuda", 0)
shapes = synth.llama_block(2048, 512, 8192)
names = ["q", "k", "v", "o", "gate", "up", "down"]
pl = usk.plan_allocation(shapes, bpw=args.bpw, rows=3, seed=0x5EED000000000003, hash="xg", layout="query")
sk = pl.new_sketch(dev)
ws = [synth.torch_weights_bf16(o, i, synth.seed_for(3, 0, k), dev) for k, (o, i) in enumerate(shapes)]
usk.build(pl, ws, sk)
usk.check(pl)
T = args.T
X = synth.torch_vector(8192, 5, dev, torch.bfloat16, T=T).reshape(-1)  # dense [T, in] views per width below
Y = torch.empty(T * 8192, dtype=torch.bfloat16, device=dev)
wsp = torch.zeros(max(usk.linear_workspace_bytes(pl, l, T) for l in range(7)), dtype=torch.uint8, device=dev)
scratch = torch.empty(8192 * 8192, dtype=torch.bfloat16, device=dev)
stream = torch.cuda.Stream(device=dev)


def timed(fn, reps=5):
    with torch.cuda.stream(stream):
        for _ in range(2):
            fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            a.record(stream)
            fn()
            b.record(stream)
        b.synchronize()
        out.append(a.elapsed_time(b))
    return sorted(out)[len(out) // 2]


rows = []
tot = {"linear": 0.0, "recon": 0.0, "cublas": 0.0}
for l, (o, i) in enumerate(shapes):
    Wd = scratch[: o * i].view(o, i)
    usk.reconstruct(pl, sk, l, Wd)
    Xl, Yl = X[:T * i].view(T, i), Y[:T * o].view(T, o)
    ms_lin = timed(lambda: usk.linear(pl, sk, l, Xl, Yl, wsp, stream=stream))
    ms_rec = timed(lambda: usk.reconstruct(pl, sk, l, Wd, stream=stream))
    Xc = Xl
    Yc = torch.empty((T, o), dtype=torch.bfloat16, device=dev)
    ms_cub = timed(lambda: torch.matmul(Xc, Wd.t(), out=Yc))
    del Xc, Yc
    fl = 2.0 * T * o * i
    r = {"linear": names[l], "out": o, "in": i, "ms_usk_linear": ms_lin, "ms_reconstruct": ms_rec,
         "ms_gemm_est": ms_lin - ms_rec, "ms_cublas": ms_cub,
         "tflops_usk": fl / ms_lin / 1e9, "tflops_gemm_est": fl / (ms_lin - ms_rec) / 1e9,
         "tflops_cublas": fl / ms_cub / 1e9}
    rows.append(r)
    tot["linear"] += ms_lin
    tot["recon"] += ms_rec
    tot["cublas"] += ms_cub
    print(json.dumps(r), flush=True)
fl = 2.0 * T * sum(o * i for o, i in shapes)
print(json.dumps({"block_total_ms": tot, "tflops_usk": fl / tot["linear"] / 1e9,
                  "tflops_cublas_dense": fl / tot["cublas"] / 1e9}), flush=True)
