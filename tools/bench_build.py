"""Build (K2) timing (tuning aid): all 112 Llama-3.2-1B linears (or the 224 Llama-3-8B-shaped ones
with --8b) in ONE usk_build call, L2 flushed before each run, median of --reps CUDA-event timings;
prints ms, weights/s, GB/s and the fraction of MEASURED_PEAKS.json HBM bandwidth."""
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
ap.add_argument("--reps", type=int, default=7)
ap.add_argument("--8b", dest="b8", action="store_true")
ap.add_argument("--hash", default="xg", choices=["x", "xg"])
ap.add_argument("--layout", default="query", choices=["query", "unit_major"])
args = ap.parse_args()
dev = torch.device("cuda", 0)
shapes = synth.llama3_8b_shapes() if args.b8 else synth.llama32_1b_shapes()
cfg = 5 if args.b8 else 3
pl = usk.plan_allocation(shapes, bpw=0.5, rows=3, seed=0x5EED000000000003, hash=args.hash,
                         layout="unit_major" if args.b8 else args.layout)
sk = pl.new_sketch(dev)
ws = [synth.torch_weights_bf16(o, i, synth.seed_for(cfg, l // 7, l % 7), dev) for l, (o, i) in enumerate(shapes)]
usk.build(pl, ws, sk)
usk.check(pl)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
t = []
for k in range(args.reps):
    flush.fill_(k)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    usk.build(pl, ws, sk)
    b.record()
    b.synchronize()
    t.append(a.elapsed_time(b))
ms = float(np.median(t))
n = sum(o * i for o, i in shapes)
gbs = n * (2 + 0.5 / 8) / (ms * 1e-3) / 1e9
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6548.2) \
    if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6548.2
print(json.dumps({"model": "8b" if args.b8 else "1b", "build_ms": ms, "weights_per_s": n / (ms * 1e-3),
                  "GB_per_s": gbs, "hbm_frac": gbs / peak, "stages_env": os.environ.get("USK_BUILD_STAGES")}))
