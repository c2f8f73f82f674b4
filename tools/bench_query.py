"""Kernel-level timing of the query kernels on the Llama-3.2-1B block shapes (tuning aid).

Times each grouped sketch-GEMV launch (q|k|v, o, gate|up, down) and the standalone reconstruct
of every block-0 linear, L2 flushed before each launch, CUDA events around the launch only.
  python tools/bench_query.py [--reps 20]
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
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--bpw", type=float, default=0.5)
ap.add_argument("--model", default="1b")
args = ap.parse_args()
dev = torch.device("cuda", 0)
shapes = synth.llama_block(2048, 512, 8192) if args.model == "1b" else synth.llama_block(4096, 1024, 14336)
pl = usk.plan_allocation(shapes, bpw=args.bpw, rows=3, seed=0x5EED000000000003)
sk = pl.new_sketch(dev)
ws = [synth.torch_weights_bf16(o, i, synth.seed_for(3, 0, k), dev) for k, (o, i) in enumerate(shapes)]
usk.build(pl, ws, sk)
usk.check(pl)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
_bt = []
for _ in range(3):
    flush.fill_(1)
    _a, _b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    _a.record()
    usk.build(pl, ws, sk)
    _b.record()
    _b.synchronize()
    _bt.append(_a.elapsed_time(_b) * 1000.0)
_nw = sum(o * i for o, i in shapes)
print(json.dumps({"build_block_us": round(min(_bt), 1), "build_Gw_s": round(_nw / min(_bt) / 1e3, 1),
                  "build_GB_s": round(_nw * 2 / min(_bt) / 1e3, 1)}))
del ws
groups = {"qkv": [0, 1, 2], "o": [3], "gate_up": [4, 5], "down": [6]}
res = {}


def timeit(fn):
    fn()
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(args.reps):
        flush.fill_(3)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(20000)
        a.record()
        fn()
        b.record()
        b.synchronize()
        tot += a.elapsed_time(b)
    return tot / args.reps * 1000.0  # us


for name, g in groups.items():
    x = synth.torch_vector(shapes[g[0]][1], 7, dev, torch.bfloat16)[0]
    ys = [torch.empty(shapes[l][0], dtype=torch.float32, device=dev) for l in g]
    w = usk.new_batch_workspace(pl, g, device=dev)
    us = timeit(lambda: usk.linear_batch(pl, sk, g, x, ys, w))
    nw = sum(shapes[l][0] * shapes[l][1] for l in g)
    res["gemv_" + name] = {"us": us, "Gw_s": nw / us / 1e3}
scratch = torch.empty(max(o * i for o, i in shapes), dtype=torch.bfloat16, device=dev)
for l, (o, i) in enumerate(shapes):
    us = timeit(lambda: usk.reconstruct(pl, sk, l, scratch[:o * i].view(o, i)))
    res[f"rec_{l}"] = {"us": us, "Gw_s": o * i / us / 1e3}
tot_gemv = sum(v["us"] for k, v in res.items() if k.startswith("gemv"))
res["gemv_block_us"] = tot_gemv
res["est_tok_s"] = 1e6 / (tot_gemv * len(shapes) / 7 * (16 if args.model == "1b" else 32))
print(json.dumps({"env_upl": os.environ.get("USK_UPL"), **{k: (round(v["us"], 2), round(v["Gw_s"], 1)) if isinstance(v, dict) else round(v, 2) for k, v in res.items()}}))

# ---------------- prefill (config 4): usk_linear with T = 2048 x 8 tokens per block-0 linear
if os.environ.get("USK_PREFILL", "1") == "1":
    T = 16384
    pre = {}
    tot_flop = tot_us = 0.0
    for l, (o, i) in enumerate(shapes):
        X = synth.torch_vector(i, 5, dev, torch.bfloat16, T=T)
        Y = torch.empty((T, o), dtype=torch.bfloat16, device=dev)
        w = usk.new_workspace(pl, l, T, device=dev)
        us = timeit(lambda: usk.linear(pl, sk, l, X, Y, w))
        fl = 2.0 * T * o * i
        pre[f"prefill_{l}"] = (round(us, 1), round(fl / us / 1e6, 1))  # us, TFLOP/s
        tot_flop += fl
        tot_us += us
        del X, Y, w
    pre["prefill_block_TFLOPs"] = round(tot_flop / tot_us / 1e6, 1)
    print(json.dumps(pre))
