"""Steady-state rate of the packed decode kernel K4p (tuning aid): one [rows, in] layer in the query
layout, a graph of `calls` back-to-back usk_linear calls (PDL-chained), weights/s per call and per SM
clock as the row count grows (large rows amortise staging, the reduce hop and the tail).
  python tools/qsteady.py [--in 2048] [--rows 8192,65536,262144]
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
ap.add_argument("--in", dest="inn", type=int, default=2048)
ap.add_argument("--rows", default="8192,32768,131072")
ap.add_argument("--calls", type=int, default=20)
ap.add_argument("--cols", type=int, default=85, help="sketch columns per unit row (bpw follows from the rows)")
args = ap.parse_args()
dev = torch.device("cuda", 0)
n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
for R in [int(r) for r in args.rows.split(",")]:
    shapes = [(R, args.inn)]
    bpw = (3 * args.cols + 0.5) * 16.0 / R  # M * N cells of 16 bits per unit of R weights
    pl = usk.plan_allocation(shapes, bpw=bpw, rows=3, seed=7, hash="xg", layout="query")
    sk = pl.new_sketch(dev)
    usk.build(pl, [synth.torch_weights_bf16(R, args.inn, 5, dev)], sk)
    x = synth.torch_vector(args.inn, 3, dev, torch.bfloat16)
    y = torch.empty((1, R), dtype=torch.float32, device=dev)
    ws = usk.new_workspace(pl, 0, device=dev)
    st = torch.cuda.Stream(device=dev)
    with torch.cuda.stream(st):
        for _ in range(3):
            usk.linear(pl, sk, 0, x, y, ws)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for _ in range(args.calls):
            usk.linear(pl, sk, 0, x, y, ws)
    g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(st):
            a.record(st)
            g.replay()
            b.record(st)
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3 / args.calls)
    us = min(ts)
    w = R * args.inn
    print(json.dumps({"rows": R, "in": args.inn, "N": int(pl.export(0)[1][0]), "us_per_call": round(us, 2), "Tweights_s": round(w / us / 1e6, 3),
                      "w_per_clk_sm": round(w / (us * 1e-6) / n_sm / 1.965e9, 2)}), flush=True)
    del g, sk, pl
