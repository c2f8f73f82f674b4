"""In-graph timeline of one decode step (tuning only): the bench.py workload (Llama-3.2-1B, 112
linears as 64 grouped sketch-GEMV launches in a CUDA graph, L2 flushed before the step), with
USK_TRACE=1 so every CTA stamps %globaltimer at start / staged / compute done / exit.

  USK_TRACE=1 python tools/trace_step.py [--reps 5] [--csv out.csv]

Prints, per launch: start (first CTA) relative to the step's first stamp, span, the gap after the
previous launch's last CTA exit, stage and compute (mean / max over CTAs), and the tail (last
compute end -> last exit); then per-group-kind means and the whole-step breakdown.
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("USK_TRACE", "1")

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2506_17255_b200 import usk  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--bpw", type=float, default=0.5)
ap.add_argument("--blocks", type=int, default=16)
ap.add_argument("--csv", default=None)
ap.add_argument("--layout", default="query", choices=["query", "unit_major"])
ap.add_argument("--npz", default=None, help="save the raw per-CTA stamps of the last replay")
args = ap.parse_args()

dev = torch.device("cuda", 0)
shapes = synth.llama32_1b_shapes()[:7 * args.blocks]
L = len(shapes)
plan = usk.plan_allocation(shapes, bpw=args.bpw, rows=3, seed=0x5EED000000000003,
                           **({"hash": "xg", "layout": "query"} if args.layout == "query" else {}))
sketch = plan.new_sketch(dev)
ws = [synth.torch_weights_bf16(o, i, synth.seed_for(3, l // 7, l % 7), dev) for l, (o, i) in enumerate(shapes)]
usk.build(plan, ws, sketch)
usk.check(plan)
del ws
groups, kinds = [], []
for b in range(L // 7):
    base = 7 * b
    groups += [[base, base + 1, base + 2], [base + 3], [base + 4, base + 5], [base + 6]]
    kinds += ["qkv", "o", "gate_up", "down"]
xs = [synth.torch_vector(shapes[g[0]][1], 1000 + gi, dev, torch.bfloat16)[0] for gi, g in enumerate(groups)]
ys = [[torch.empty(shapes[l][0], dtype=torch.float32, device=dev) for l in g] for g in groups]
wsg = [usk.new_batch_workspace(plan, g, device=dev) for g in groups]
stream = torch.cuda.Stream(device=dev)


def step():
    for gi, g in enumerate(groups):
        usk.linear_batch(plan, sketch, g, xs[gi], ys[gi], wsg[gi])


with torch.cuda.stream(stream):
    step()
    step()
torch.cuda.synchronize()
usk.trace_reset()
graph = torch.cuda.CUDAGraph()
with torch.cuda.graph(graph, stream=stream):
    step()
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ms = []
for r in range(args.reps):
    with torch.cuda.stream(stream):
        flush.fill_(r & 0xFF)
        ev[0].record(stream)
        graph.replay()
        ev[1].record(stream)
    torch.cuda.synchronize()
    ms.append(ev[0].elapsed_time(ev[1]))
tr = usk.trace_read()
per = len(tr) // len(groups)  # launches per group (compute [+ reduce])
assert per * len(groups) == len(tr), (len(tr), len(groups))
kinds = [k + ("" if j == 0 else f".{j}") for k in kinds for j in range(per)]
t0 = min(int(t[:, 0].min()) for t in tr)
rows = []
prev_end = t0
for k, t in enumerate(tr):
    st, sg, cd, ex = (t[:, c] - t0 for c in range(4))
    start, end = int(st.min()), int(ex.max())
    rows.append(dict(k=k, kind=kinds[k], grid=t.shape[0], start=start / 1e3, span=(end - start) / 1e3,
                     gap=(start - (prev_end - t0)) / 1e3, stage=float((sg - st).mean()) / 1e3,
                     stage_max=float((sg - st).max()) / 1e3, comp=float((cd - sg).mean()) / 1e3,
                     comp_max=float((cd - sg).max()) / 1e3, first_comp=float(sg.min() - start) / 1e3,
                     tail=float(ex.max() - cd.max()) / 1e3, skew=float(st.max() - st.min()) / 1e3))
    prev_end = end + t0
step_us = (prev_end - t0) / 1e3
print(f"graph replay (events): {np.median(ms) * 1e3:.1f} us   traced step span: {step_us:.1f} us")
hdr = ("k", "kind", "grid", "start", "span", "gap", "skew", "stage", "stage_max", "first_comp", "comp", "comp_max", "tail")
print(" ".join(f"{h:>9}" for h in hdr))
for r in rows[:4 * per] + rows[-2 * per:]:
    print(" ".join(f"{r[h]:>9.2f}" if isinstance(r[h], float) else f"{r[h]:>9}" for h in hdr))
print("per kind (mean over blocks):")
for kd in dict.fromkeys(kinds):
    sel = [r for r in rows if r["kind"] == kd]
    print(f"  {kd:8s} grid={sel[0]['grid']:4d} " + " ".join(
        f"{h}={np.mean([r[h] for r in sel]):.2f}" for h in ("span", "gap", "skew", "stage", "stage_max", "comp", "comp_max", "tail")))
spans = sum(r["span"] for r in rows)
gaps = sum(max(0.0, r["gap"]) for r in rows)
overl = sum(min(0.0, r["gap"]) for r in rows)
comp = sum(r["comp"] for r in rows)
print(f"sum spans {spans:.1f} us, sum gaps {gaps:.1f} us (overlap {overl:.1f}), sum mean-compute {comp:.1f} us, "
      f"step {step_us:.1f} us")
# critical path per grouped call: previous reduce end -> first CTA past its wait (release + x load),
# CTA compute starts spread (staging exposed after the release), compute (first start -> last compute
# end), last compute end -> this call's reduce end (the reduce hop)
if per == 2:
    cp = {"release": [], "start_spread": [], "compute": [], "hop": [], "comp_mean": []}
    sub = {"issue": [], "land": [], "convert": [], "wait": [], "x": []}  # mean per-CTA stage phases
    for g in range(1, len(groups)):
        tc, trd, tprev = tr[2 * g], tr[2 * g + 1], tr[2 * g - 1]
        r_prev = int(tprev[:, 3].max())
        sg = tc[:, 1].astype(np.int64)
        cd = tc[:, 2].astype(np.int64)
        cp["release"].append((sg.min() - r_prev) / 1e3)
        cp["start_spread"].append((sg.max() - sg.min()) / 1e3)
        cp["compute"].append((cd.max() - sg.max()) / 1e3)
        cp["comp_mean"].append(float((cd - sg).mean()) / 1e3)
        cp["hop"].append((int(trd[:, 3].max()) - cd.max()) / 1e3)
        st0, iss, lnd, cvt, wtd = (tc[:, c].astype(np.int64) for c in (0, 4, 5, 6, 7))
        sub["issue"].append(float((iss - st0).mean()) / 1e3)
        sub["land"].append(float((lnd - iss).mean()) / 1e3)
        sub["convert"].append(float((cvt - lnd).mean()) / 1e3)
        sub["wait"].append(float((wtd - cvt).mean()) / 1e3)
        sub["x"].append(float((sg - wtd).mean()) / 1e3)
    print("critical path per call (us, mean over calls 1..):", " ".join(f"{k}={np.mean(v):.2f}" for k, v in cp.items()))
    for kd in ("qkv", "o", "gate_up", "down"):
        idx = [g - 1 for g in range(1, len(groups)) if groups and kinds[2 * g] == kd]
        print(f"  {kd:8s}", " ".join(f"{k}={np.mean([v[i] for i in idx]):.2f}" for k, v in cp.items()),
              f"sum={np.mean([cp['release'][i] + cp['start_spread'][i] + cp['compute'][i] + cp['hop'][i] for i in idx]):.2f}")
        print(f"  {'':8s} stage phases (CTA mean):", " ".join(f"{k}={np.mean([v[i] for i in idx]):.2f}" for k, v in sub.items()))
if args.npz:
    np.savez(args.npz, **{f"l{k}": t for k, t in enumerate(tr)}, kinds=np.array(kinds))
if args.csv:
    import csv
    with open(args.csv, "w", newline="") as f:
        w = csv.DictWriter(f, fieldnames=list(rows[0].keys()))
        w.writeheader()
        w.writerows(rows)
