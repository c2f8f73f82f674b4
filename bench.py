#!/usr/bin/env python
"""Benchmark of the B200-native UltraSketchLLM sketch hot path (BASELINE.json metric).

Workload (BASELINE.json configs[2], "c3"): Llama-3.2-1B, all 112 linear layers (16 blocks x
q,k,v,o,gate,up,down), synthetic random bf16 weights (synth recipe), ROW granularity, M = 3 rows,
0.5 bits per weight, uniform importance.  One STEP = one batch-1 decode token = the 112 fused
sketch-GEMV launches (usk_linear, T = 1) in model order, replayed as one CUDA graph.  L2 is
flushed (256 MB write) before every timed step, so the 60.8 MB sketch is re-read from HBM.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl usk|reference]

N > 1 (one rank per GPU, NCCL): `--gpus N` spawns the N ranks itself (torch.distributed.run on
127.0.0.1) unless it already runs under a launcher, whose WORLD_SIZE must equal N.  Every linear's
output features are sharded over the ranks; the y shards of a grouped call (q|k|v, o, gate|up,
down) land in one contiguous per-rank buffer and are all-gathered with ONE NCCL collective per call
(64 per token), captured in the step's CUDA graph (strong scaling).  --dist-selftest runs the same
launcher and host logic on CPU (gloo) with synthetic shard outputs: the CPU test of the N > 1 path.
--impl reference times the CPU oracle (oracle/, plain C) on a bounded sample of the same
workload, on rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "fused sketch-GEMV decode tokens/s + weights reconstructed/s, Llama-3.2-1B @0.5 bpw"
UNIT = "tokens/s"
BPW, ROWS, SEED = 0.5, 3, 0x5EED000000000003
CFG = 3  # synth seed namespace (BASELINE.json configs[2])


def _peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0, "_fallback": True}


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi sampling (every 50 ms) DURING the timed region: one persistent process."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.FIELDS,
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.3)  # let the first sample land inside the region
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is None:
            return
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=10)
        except Exception:
            self.proc.kill()
            out = ""
        for line in (out or "").splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) >= 8:
                self.samples.append(f)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        num = lambda v: float(v) if v.replace(".", "", 1).isdigit() else None
        sm = [num(s[0]) for s in self.samples if num(s[0]) is not None]
        mx = [num(s[1]) for s in self.samples if num(s[1]) is not None]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for s in self.samples:
            for k, n in enumerate(names):
                if s[4 + k].lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.samples)}


# ----------------------------------------------------------------------------- CPU oracle leg
def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


_ORACLE_CTX = {}


def oracle_decode_sample(shapes, weights_for_layer, budget_s=12.0, threads=1, rows_per_call=32):
    """Time the CPU oracle's fp64 sketch-GEMV (reconstruct-on-the-fly + FMA, oracle/usk_oracle.c, as
    it stands) on a bounded sample: the 7 linears of block 0, output rows in round-robin until
    ~budget_s of wall time has run.  threads > 1: that many host threads call the oracle at once on
    disjoint row slices (ctypes releases the GIL during each C call; OpenMP-free, every core busy).
    Returns tokens/s extrapolated by weights/s over all 112 linears."""
    import concurrent.futures as cf

    import oracle
    blk = shapes[:7]
    # the oracle's block-0 plan and sketch are built once per process (the timed sample is the GEMV)
    key = (tuple(blk), id(weights_for_layer))
    if _ORACLE_CTX.get("key") != key:
        opl = oracle.plan(blk, BPW, M=ROWS, dtype=oracle.BF16, seed=SEED)
        sk = np.zeros(opl.total_cells, np.uint16)
        for l in range(7):
            oracle.build_layer(opl, l, weights_for_layer(l), sk)
        xs = [synth.vector(i, seed=1000 + l)[0].astype(np.float64) for l, (o, i) in enumerate(blk)]
        _ORACLE_CTX.update(key=key, opl=opl, sk=sk, xs=xs)
    opl, sk, xs = _ORACLE_CTX["opl"], _ORACLE_CTX["sk"], _ORACLE_CTX["xs"]
    RS = rows_per_call  # output rows per oracle call

    def worker(k):
        done, row = 0, k
        t_end = time.perf_counter() + budget_s
        while time.perf_counter() < t_end:
            for l, (o, i) in enumerate(blk):
                r0 = (row * RS) % o
                oracle.linear_rows(opl, sk, l, xs[l], r0, r0 + RS)
                done += RS * i
            row += threads
        return done

    t0 = time.perf_counter()
    with cf.ThreadPoolExecutor(max_workers=threads) as ex:
        done_w = sum(ex.map(worker, range(threads)))
    spent = time.perf_counter() - t0
    wps = done_w / spent
    total_w = sum(o * i for o, i in shapes)
    return {"value": wps / total_w, "unit": UNIT, "cores": threads, "kind": "oracle",
            "sample": f"oracle fp64 sketch-GEMV of {done_w} weights ({RS}-row slices of the 7 block-0 linears, "
                      f"{spent:.1f} s wall on {threads} host thread(s)), extrapolated to the 112-linear token by "
                      f"weights/s",
            "host": {"cpu_model": _cpu_model(), "os_cpu_count": os.cpu_count(),
                     "OMP_NUM_THREADS": os.environ.get("OMP_NUM_THREADS")},
            "weights_per_s": wps}


def host_block0_weights(shapes):
    import torch
    def get(l):
        o, i = shapes[l]
        w = synth.torch_weights_bf16(o, i, synth.seed_for(CFG, 0, l), "cuda")
        return w.cpu().view(torch.int16).numpy().view(np.uint16).copy()
    return get


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import torch
    shapes = synth.llama32_1b_shapes()
    if torch.cuda.is_available():
        getw = host_block0_weights(shapes)
    else:
        getw = lambda l: synth.weights_bf16(shapes[l][0], shapes[l][1], synth.seed_for(CFG, 0, l))
    per_step = []
    # the whole --steps K --warmup W run samples ~60 s of oracle work (each step a bounded sample of
    # the same workload, >= 0.2 s), after one build of the oracle's block-0 sketch
    budget = args.ref_step_s if args.ref_step_s else max(0.2, 60.0 / max(1, args.steps + args.warmup))
    ncores = max(1, len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count() or 1)
    for k in range(args.warmup + args.steps):
        r = oracle_decode_sample(shapes, getw, budget_s=budget, threads=ncores)  # the box's host cores
        if k >= args.warmup:
            per_step.append(r)
    v = float(np.mean([r["value"] for r in per_step]))
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 / v, "higher_is_better": True,
            "scaling": "strong" if args.gpus > 1 else "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "c3: Llama-3.2-1B 112 linears, batch-1 decode, 0.5 bpw, M=3, bf16 weights",
                       "bpw": BPW, "rows": ROWS},
            "cpu_baseline": {**{k: per_step[-1][k] for k in ("kind", "cores", "sample")}, "value": v, "unit": UNIT},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- GPU leg
def run_usk(args):
    import torch
    import torch.distributed as dist
    from paper_2506_17255_b200 import dist as udist
    from paper_2506_17255_b200 import usk

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    peaks = _peaks()
    shapes = synth.llama32_1b_shapes()
    L = len(shapes)
    numel = sum(o * i for o, i in shapes)

    # ---- plan + build (layer-sharded across ranks, then a one-time replication of the sketch)
    # the headline plan: USK-XG unit keys (ledger L32) in the query layout (usk.h USK_LAYOUT_QUERY,
    # packed decode kernels K4p/K3p); --layout unit_major times the round-1 plan (USK-X, K4)
    LAY = {"query": dict(hash="xg", layout="query"), "unit_major": dict(hash="x", layout="unit_major")}[args.layout]
    plan = usk.plan_allocation(shapes, bpw=BPW, rows=ROWS, seed=SEED, **LAY)
    sketch = plan.new_sketch(dev)
    sketch.zero_()
    owned = udist.owned_layers(L, rank, world)  # whole blocks round-robin over ranks
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # all owned layers in ONE usk_build call (the kernel balances its tiles across waves); the
    # weights (1.95 GB bf16 for all 112 linears) are generated first and freed after the build
    ws = [synth.torch_weights_bf16(shapes[l][0], shapes[l][1], synth.seed_for(CFG, l // 7, l % 7), dev) for l in owned]
    usk.build(plan, ws, sketch, layer_ids=owned)  # warm-up (module load, attributes)
    build_times = []
    for _ in range(7):
        flush_b = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
        flush_b.fill_(1)
        del flush_b
        torch.cuda.synchronize()
        ev0.record()
        usk.build(plan, ws, sketch, layer_ids=owned)
        ev1.record()
        torch.cuda.synchronize()
        build_times.append(ev0.elapsed_time(ev1))
    build_ms = float(np.median(build_times))
    del ws
    usk.check(plan)
    owned_w = sum(shapes[l][0] * shapes[l][1] for l in owned)
    replicate_ms = 0.0
    if world > 1:  # one-time replication of the layer-sharded sketch (deployment step)
        if args.layout == "query":
            regions = [(plan.layers[l].qbyte_begin, plan.layers[l].qbyte_begin + plan.layers[l].qbytes) for l in range(L)]
        else:
            regions = [(plan.layers[l].cell_begin * 2, (plan.layers[l].cell_begin + plan.layers[l].n_cells) * 2)
                       for l in range(L)]
        torch.cuda.synchronize()
        ev0.record()
        udist.replicate_sketch(sketch, regions, world)
        ev1.record()
        torch.cuda.synchronize()
        replicate_ms = ev0.elapsed_time(ev1)

    # ---- decode buffers.  The linears of a block that read the same activation share one
    #      synthetic x (q|k|v: attention input, o, gate|up: MLP input, down), exactly as in a
    #      decode step; y is fp32.  Grouped launches (usk_linear_batch): 4 per block = 64/token.
    def shard(o):
        return udist.output_shard(o, rank, world)
    groups = []
    for b in range(L // 7):
        base = 7 * b
        groups += [[base, base + 1, base + 2], [base + 3], [base + 4, base + 5], [base + 6]]
    xin = [shapes[g[0]][1] for g in groups]
    x_off = np.cumsum([0] + xin)
    out_off = np.cumsum([0] + [o for o, i in shapes])
    X = torch.empty(int(x_off[-1]), dtype=torch.bfloat16, device=dev)
    for gi, g in enumerate(groups):
        X[x_off[gi]:x_off[gi + 1]] = synth.torch_vector(xin[gi], 1000 + gi, dev, torch.bfloat16)[0]
    Y = torch.zeros(int(out_off[-1]), dtype=torch.float32, device=dev)
    xg = [X[x_off[gi]:x_off[gi + 1]] for gi in range(len(groups))]
    x_of_layer = {l: xg[gi] for gi, g in enumerate(groups) for l in g}
    ys_full = [Y[out_off[l]:out_off[l + 1]] for l in range(L)]
    ranges = {l: shard(shapes[l][0]) for l in range(L)}
    # N > 1: a group's y shards live in one contiguous buffer, gathered by one collective per call
    glay = [udist.group_shard_layout([shapes[l][0] for l in g], rank, world) for g in groups]
    Gsh = [torch.zeros(pad, dtype=torch.float32, device=dev) for _, pad in glay]
    g_off = np.cumsum([0] + [world * pad for _, pad in glay])
    GF = torch.zeros(int(g_off[-1]), dtype=torch.float32, device=dev)   # every group's gathered y, one buffer
    Gfull = [GF[g_off[gi]:g_off[gi + 1]] for gi in range(len(groups))]
    Yshard = {}
    for gi, g in enumerate(groups):
        for k, l in enumerate(g):
            o0, o1, off = glay[gi][0][k]
            Yshard[l] = Gsh[gi][off:off + (o1 - o0)]
    ws_group = [usk.new_batch_workspace(plan, g, [ranges[l] for l in g], device=dev) for g in groups]
    ws_layer = [usk.new_workspace(plan, l, 1, *ranges[l], device=dev) for l in range(L)]
    out_of = (lambda l: ys_full[l]) if world == 1 else (lambda l: Yshard[l])

    group_of = {l: gi for gi, g in enumerate(groups) for l in g}

    peer_bufs = None
    if world > 1 and args.collective == "peer":  # fused y all-gather in the reduce kernel (symmetric memory)
        peer_bufs = udist.PeerYBuffers(usk, [[shapes[l][0] for l in g] for g in groups], dev)
        ws_peer = [usk.new_batch_workspace(plan, g, [ranges[l] for l in g], device=dev) for g in groups]

    def gather(ls):  # one all-gather per grouped call (per linear for the 112-launch variant)
        if world > 1:
            gi = group_of[ls[0]]
            if len(ls) == len(groups[gi]):
                udist.allgather_group(Gsh[gi], Gfull[gi])
            else:
                for l in ls:
                    udist.allgather_outputs(Yshard[l].contiguous(), ys_full[l])

    def warm():
        if args.prefetch:  # opt-in: the step reads the whole sketch (60 MB < L2) from HBM once, up front
            usk.prefetch_l2(plan, sketch)

    def step_grouped():
        warm()
        for gi, g in enumerate(groups):
            if args.prefetch_next and gi + 1 < len(groups):  # L2 hint: the next group's sketch + metadata
                usk.prefetch_l2(plan, sketch, groups[gi + 1][0], groups[gi + 1][-1] + 1)
            if peer_bufs is not None:
                usk.linear_batch_peers(plan, sketch, g, xg[gi], peer_bufs.peers(gi), ws_peer[gi],
                                       ranges=[ranges[l] for l in g])
                usk.peer_wait(plan, peer_bufs.peers(gi))
                continue
            usk.linear_batch(plan, sketch, g, xg[gi], [out_of(l) for l in g], ws_group[gi],
                             ranges=[ranges[l] for l in g])
            gather(g)

    def step_single():
        warm()
        for l in range(L):
            usk.linear(plan, sketch, l, x_of_layer[l].view(1, -1), out_of(l).view(1, -1), ws_layer[l], *ranges[l])
            gather([l])

    stream = torch.cuda.Stream(device=dev)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)  # > 126 MB L2

    def capture(fn):
        if world > 1 and os.environ.get("USK_BENCH_NCCL_GRAPH") == "0":  # opt-out: eager steps
            torch.cuda.synchronize()
            usk.launch_count(reset=True)
            with torch.cuda.stream(stream):
                fn()
            torch.cuda.synchronize()
            return None, usk.launch_count(reset=True)  # eager steps (NCCL in graph capture is opt-in)
        torch.cuda.synchronize()
        with torch.cuda.stream(stream):
            for _ in range(2):
                fn()  # warm (module load, smem attributes) before capture
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        usk.launch_count(reset=True)
        try:
            with torch.cuda.graph(g, stream=stream):
                fn()
            return g, usk.launch_count(reset=True)
        except Exception as e:  # NCCL capture unsupported -> eager steps
            print(f"[bench] graph capture failed ({e}); timing eager steps", file=sys.stderr)
            return None, usk.launch_count(reset=True)

    def replay(g, fn):
        if g is not None:
            g.replay()
        else:
            with torch.cuda.stream(stream):
                fn()

    def time_steps(g, fn, steps, warmup, clocks=None):
        for _ in range(max(3, warmup)):
            replay(g, fn)
        torch.cuda.synchronize()
        starts = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
        ends = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        for k in range(steps):
            with torch.cuda.stream(stream):
                flush.fill_(k & 0xFF)          # untimed L2 flush
                starts[k].record(stream)
                replay(g, fn)
                ends[k].record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        total = float(sum(s.elapsed_time(e) for s, e in zip(starts, ends)))
        if world > 1:
            t = torch.tensor([total], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            total = float(t.item())
        return total / steps

    g_grp, launches_grp = capture(step_grouped)
    g_one, launches_one = capture(step_single)
    def full_y():  # the step's outputs in layer order (N > 1: assembled from the gathered buffers)
        if world == 1:
            return Y.clone()
        if peer_bufs is not None:
            return torch.cat([t for yg in peer_bufs.y for t in yg])
        ys = []
        for gi, g in enumerate(groups):
            ys += udist.assemble_group(Gfull[gi], [shapes[l][0] for l in g], world)
        return torch.cat(ys)

    y_check = None
    with ClockSampler(local) as clocks:
        ms_per_step = time_steps(g_grp, step_grouped, args.steps, args.warmup)
        y_check = full_y()
        ms_single = time_steps(g_one, step_single, args.steps, args.warmup)
    same = bool(torch.equal(y_check, Y))   # grouped and per-linear launches give identical bits
    import hashlib
    y_sha = hashlib.sha256(y_check.cpu().numpy().tobytes()).hexdigest()[:16]  # equal for every N
    use_graph = g_grp is not None
    launches_per_step = launches_grp
    tok_s = 1000.0 / ms_per_step

    # ---- per-launch kernel durations (same launches, eager, each bracketed by events behind a
    #      GPU sleep so the host enqueue latency is hidden) -> roofline of the dominant kernel
    kern_ms = np.zeros(len(groups))
    reps = 5
    with torch.cuda.stream(stream):
        for rep in range(reps):
            for gi, g in enumerate(groups):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda._sleep(20000)
                a.record(stream)
                usk.linear_batch(plan, sketch, g, xg[gi], [out_of(l) for l in g], ws_group[gi],
                                 ranges=[ranges[l] for l in g], stream=stream)
                b.record(stream)
                b.synchronize()
                kern_ms[gi] += a.elapsed_time(b) / reps
    w_rank = sum((shard(o)[1] - shard(o)[0]) * i for o, i in shapes)
    sum_kern = float(kern_ms.sum())
    clk = clocks.summary()
    f_peak = float(peaks.get("sm_max_mhz", 1965.0)) * 1e6
    n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
    # Roofline of the sketch query: the method gathers M = 3 cells per
    # weight and token from shared memory.  The floor is the shared-memory bandwidth, 128 B/clk/SM:
    #  * query layout (K4p): 2-byte cells, a key group's 8 cells in one 16-B load -> 64 / M weight/clk/SM
    #  * unit-major layout (K4): one 32-bit word per lookup -> 32 / M weight/clk/SM
    # The design-dependent instruction-issue line is reported beside it (per 256 weights of a warp in
    # K4p: LDS.128 of R + 3 x (LOP3 + FFMA.RZ + IMAD + LDS.128) + 4 VIMNMX3.U16x2 + 4 x (SHF + SHL +
    # LOP3) + 8 FHFMA.BF16 = 37; in K4: 14 per 32 weights)
    QL = args.layout == "query"
    ISSUE = 37.0 / 8 if QL else 14.0
    alu_peak = n_sm * 4 * 32 / ISSUE * f_peak / 1e9             # Gweight/s
    per_clk = (128.0 / (2 * ROWS)) if QL else 32.0 / ROWS
    gather_floor = n_sm * per_clk * f_peak / 1e9                 # Gweight/s
    # the timed graph holds only the sketch-GEMV launches (k_gemv_fast + k_gemv_reduce per group),
    # so their achieved rate over the timed region is the step's weights / step time
    achieved = w_rank / (ms_per_step * 1e-3) / 1e9
    sketch_bytes = plan.info["total_cells"] * 2
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        traffic = json.load(open(tp)).get("k_qgemv_bytes_per_launch" if QL else "k_gemv_fast_bytes_per_launch")

    # ---- standalone reconstruct throughput (weights reconstructed/s, HBM-bound kernel): the 112
    #      layer reconstructions into one scratch buffer, captured as one CUDA graph, L2 flushed
    # query layout: usk_reconstruct_batch, each block's q|k|v|o|gate|up in one K3p launch (in = 2048)
    # and down in another, every layer into its own region of a block-sized scratch
    blk = shapes[:7]
    scratch = torch.empty(sum(o * i for o, i in blk), dtype=torch.bfloat16, device=dev)
    soff = np.cumsum([0] + [o * i for o, i in blk])
    souts = [scratch[soff[k]:soff[k + 1]].view(o, i) for k, (o, i) in enumerate(blk)]

    def rec_all():
        if args.layout == "query":
            for b in range(L // 7):
                usk.reconstruct_batch(plan, sketch, list(range(7 * b, 7 * b + 7)), souts, stream=stream)
            return
        for l, (o, i) in enumerate(shapes):
            usk.reconstruct(plan, sketch, l, souts[l % 7], stream=stream)

    with torch.cuda.stream(stream):
        rec_all()
    torch.cuda.synchronize()
    g_rec = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g_rec, stream=stream):
        rec_all()
    rec_runs = []
    for k in range(5):
        with torch.cuda.stream(stream):
            flush.fill_(k & 0xFF)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            g_rec.replay()
            b.record(stream)
        b.synchronize()
        rec_runs.append(a.elapsed_time(b))
    rec_ms = float(np.median(rec_runs))
    rec_wps = numel / (rec_ms * 1e-3)

    # ---- end-to-end through the binding: pinned host x -> device, 112 linears, y -> pinned host
    Xh = X.cpu().pin_memory()
    Yout = Y if world == 1 else (peer_bufs.yflat if peer_bufs is not None else GF)  # what the step leaves
    Yh = torch.empty(Yout.numel(), dtype=torch.float32).pin_memory()
    g2 = torch.cuda.CUDAGraph()
    e2e_graph = True
    try:
        with torch.cuda.graph(g2, stream=stream):
            X.copy_(Xh, non_blocking=True)
            step_grouped()
            Yh.copy_(Yout, non_blocking=True)
    except Exception:
        e2e_graph = False
    e_ms = []
    for k in range(max(3, args.warmup) + args.steps):
        with torch.cuda.stream(stream):
            flush.fill_(2)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            if e2e_graph:
                g2.replay()
            else:
                X.copy_(Xh, non_blocking=True)
                step_grouped()
                Yh.copy_(Yout, non_blocking=True)
            b.record(stream)
        b.synchronize()
        if k >= max(3, args.warmup):
            e_ms.append(a.elapsed_time(b))
    e2e_copy_ms = float(np.mean(e_ms))
    # the same step with the reduce kernels storing y straight into the pinned host buffer (zero-copy:
    # the D2H transfer is the kernels' own PCIe writes, complete when the step's stream is), the x
    # H2D copy kept: the usk_linear_batch outputs are host-mapped views of Yh (UVA)
    e2e_zc_ms = None
    if world == 1 and e2e_graph:
        Yhz = torch.empty(Y.numel(), dtype=torch.float32).pin_memory()
        yz = [Yhz[out_off[l]:out_off[l + 1]] for l in range(L)]

        def step_zc():
            for gi, g in enumerate(groups):
                usk.linear_batch(plan, sketch, g, xg[gi], [yz[l] for l in g], ws_group[gi])

        try:
            g3 = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g3, stream=stream):
                X.copy_(Xh, non_blocking=True)
                step_zc()
            z_ms = []
            for k in range(max(3, args.warmup) + args.steps):
                with torch.cuda.stream(stream):
                    flush.fill_(2)
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record(stream)
                    g3.replay()
                    b.record(stream)
                b.synchronize()
                if k >= max(3, args.warmup):
                    z_ms.append(a.elapsed_time(b))
            if torch.equal(Yhz, Yh):  # the same bits as the copy-back variant
                e2e_zc_ms = float(np.mean(z_ms))
            del g3
        except Exception as e:  # pragma: no cover - reported, the copy variant stays
            print(f"[bench] zero-copy e2e failed ({e})", file=sys.stderr)
    e2e_ms = min(e2e_copy_ms, e2e_zc_ms) if e2e_zc_ms is not None else e2e_copy_ms
    if world > 1:
        t = torch.tensor([e2e_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())

    # ---- extra plans on the same workload and grouping, measured the same way:
    #      * the paper's own 0.5-bpw point: a 1/8-rate sketch of 4-bit states (Table 1 "+ q4",
    #        SURVEY 8(f1)), q4 plan (G = 128);
    #      * importance-aware allocation with per-class rows (ledger L30): C = 4
    #        saliency classes (synth recipe), class rows (3, 3, 2, 2)
    def extra_point(**kw):
        try:
            return extra_point_(**kw)
        except usk.UskError as e:  # a plan the library refuses is reported, the headline line stays
            print(f"[bench] extra point {kw.get('layout', '')} failed: {e}", file=sys.stderr)
            return {"error": str(e)}

    def extra_point_(**kw):
        xplan = usk.plan_allocation(shapes, bpw=BPW, rows=ROWS, seed=SEED, **kw)
        xsk = xplan.new_sketch(dev)
        wq = [synth.torch_weights_bf16(shapes[l][0], shapes[l][1], synth.seed_for(CFG, l // 7, l % 7), dev)
              for l in range(L)]
        usk.build(xplan, wq, xsk)
        torch.cuda.synchronize()
        ev0.record()
        usk.build(xplan, wq, xsk)
        ev1.record()
        torch.cuda.synchronize()
        xbuild_ms = ev0.elapsed_time(ev1)
        del wq
        usk.check(xplan)
        ws_x = [usk.new_batch_workspace(xplan, g, device=dev) for g in groups]

        def step_x():
            for gi, g in enumerate(groups):
                usk.linear_batch(xplan, xsk, g, xg[gi], [ys_full[l] for l in g], ws_x[gi])

        gx, lx = capture(step_x)
        xms = time_steps(gx, step_x, max(20, args.steps // 4), args.warmup)
        return {"tokens_per_s": 1000.0 / xms, "ms_per_step": xms, "sketch_MB": xplan.sketch_bytes / 1e6,
                "cells": xplan.info["total_cells"], "achieved_bpw": xplan.info["achieved_bits"] / xplan.info["numel"],
                "build_ms": xbuild_ms, "launches_per_step": lx}

    def paper_six_of_seven():
        """The paper's own configuration (ledger L14): Q, K, V, Up, Down, Gate sketched,
        O kept dense -- each block's o projection as a bf16 cuBLAS GEMV (torch.mv) in the same graph."""
        nb = L // 7
        Wo = [synth.torch_weights_bf16(shapes[7 * b + 3][0], shapes[7 * b + 3][1], synth.seed_for(CFG, b, 3), dev)
              for b in range(nb)]
        yo = [torch.empty(shapes[7 * b + 3][0], dtype=torch.bfloat16, device=dev) for b in range(nb)]

        def step67():
            for gi, g in enumerate(groups):
                if len(g) == 1 and g[0] % 7 == 3:
                    torch.mv(Wo[g[0] // 7], xg[gi], out=yo[g[0] // 7])
                else:
                    usk.linear_batch(plan, sketch, g, xg[gi], [ys_full[l] for l in g], ws_group[gi])

        g67, l67 = capture(step67)
        ms67 = time_steps(g67, step67, max(20, args.steps // 4), args.warmup)
        sk_w = sum(o * i for l, (o, i) in enumerate(shapes) if l % 7 != 3)
        del Wo, yo, g67
        return {"tokens_per_s": 1000.0 / ms67, "ms_per_step": ms67, "sketched_linears": L - nb,
                "dense": "o projection, bf16 weights, torch.mv (cuBLAS GEMV)", "sketched_weights": sk_w,
                "launches_per_step_usk": l67}

    q4 = cls = orow = p67 = um = None
    if world == 1 and not args.no_q4:
        del g_rec, g2
        torch.cuda.empty_cache()
        if args.layout == "query":  # the round-1 plan on the same workload: USK-X keys, unit-major K4
            um = extra_point(hash="x", layout="unit_major")
            um.update({"hash": "USK-X (one key per unit)", "layout": "unit_major", "kernels": "k_gemv_fast + k_gemv_reduce"})
            torch.cuda.empty_cache()
        q4 = extra_point(state_bits=4, group_size=128)
        q4.update({"state_bits": 4, "group_size": 128})
        torch.cuda.empty_cache()
        sal = [torch.from_numpy(synth.saliency_like(i, 500 + l)).to(dev) for l, (o, i) in enumerate(shapes)]
        # USK-XG keys, classes scored per key group (ledger L33): one N per group; in the query layout
        # the key groups are in class order, the top class of gate/up in 64-unit chunks (ledger L34)
        ckw = {"hash": "xg", "layout": "query"} if args.layout == "query" else {}
        cls = extra_point(saliency=sal, n_classes=4, class_rows=(3, 3, 2, 2), **ckw)
        cls.update({"n_classes": 4, "class_rows": [3, 3, 2, 2], "saliency": "synth.saliency_like (log-normal, 1% of dims x400)",
                    "hash": "USK-XG (classes per key group, ledger L33)" if ckw else "USK-X",
                    "layout": ckw.get("layout", "unit_major")})
        torch.cuda.empty_cache()
        orow = extra_point(granularity="outrow")
        orow.update({"granularity": "outrow (one unit per output row, ledger L31)"})
        torch.cuda.empty_cache()
        p67 = paper_six_of_seven()

    # ---- BASELINE config 4: Llama-3.2-1B prefill, 2048 tokens x batch 8 (T = 16384) through all 112
    #      linears in model order, grouped as the decode (usk_linear_batch_tokens: K3 reconstruct of the
    #      group into the workspace + one tcgen05 GEMM K5), at 0.5 bpw (the decode plan) and 0.8 bpw;
    #      X/Y (268+ MB each) exceed L2
    c4 = None
    if world == 1 and not args.no_prefill:
        torch.cuda.empty_cache()
        T = 16384
        Xp = synth.torch_vector(8192, 77, dev, torch.bfloat16, T=T).reshape(-1)  # T x 8192 bf16 N(0,1)
        gout = max(sum(shapes[l][0] for l in g) for g in groups)
        Yp = torch.empty(T * gout, dtype=torch.bfloat16, device=dev)
        # dense row-major [T, in] / [T, out] per layer (the T > 1 layout; the binding rejects strided
        # views); a group's outputs are consecutive [T, out_k] blocks of Yp
        Xw = {i: Xp[:T * i].view(T, i) for i in {i for _, i in shapes}}
        Yw = {o: Yp[:T * o].view(T, o) for o in {o for o, _ in shapes}}

        def group_ys(g):
            ys, off = [], 0
            for l in g:
                ys.append(Yp[off:off + T * shapes[l][0]].view(T, shapes[l][0]))
                off += T * shapes[l][0]
            return ys

        Yg = [group_ys(g) for g in groups]
        ws_p = torch.zeros(max(max(usk.linear_workspace_bytes(plan, l, T) for l in range(L)),
                               max(usk.linear_batch_tokens_workspace_bytes(plan, g, T) for g in groups)),
                           dtype=torch.uint8, device=dev)

        def prefill_pass(pl_, sk_):
            # per group (q|k|v, o, gate|up, down): the group's W' rebuilt once into the workspace,
            # then one tcgen05 GEMM writing each layer's Y (usk_linear_batch_tokens)
            for gi, g in enumerate(groups):
                usk.linear_batch_tokens(pl_, sk_, g, Xw[shapes[g[0]][1]], Yg[gi], ws_p, stream=stream)

        def prefill_pass_single(pl_, sk_):
            for l, (o, i) in enumerate(shapes):
                usk.linear(pl_, sk_, l, Xw[i], Yw[o], ws_p, stream=stream)

        def time_pass(pl_, sk_, reps=7, graph=True, fn=prefill_pass):
            # the launches of a pass captured in one CUDA graph, as the decode step (eager timing is
            # reported beside); median of single passes (X, Y and the workspace exceed L2 anyway)
            with torch.cuda.stream(stream):
                fn(pl_, sk_)
            torch.cuda.synchronize()
            gp = None
            if graph:
                gp = torch.cuda.CUDAGraph()
                with torch.cuda.graph(gp, stream=stream):
                    fn(pl_, sk_)
            ts = []
            for _ in range(reps):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                with torch.cuda.stream(stream):
                    a.record(stream)
                    gp.replay() if gp is not None else fn(pl_, sk_)
                    b.record(stream)
                b.synchronize()
                ts.append(a.elapsed_time(b))
            del gp
            return float(np.median(ts))

        flop = 2.0 * T * numel
        ms05 = time_pass(plan, sketch)
        ms05_eager = time_pass(plan, sketch, graph=False)
        ms05_single = time_pass(plan, sketch, fn=prefill_pass_single)
        plan08 = usk.plan_allocation(shapes, bpw=0.8, rows=ROWS, seed=SEED, **LAY)
        sk08 = plan08.new_sketch(dev)
        w8_ = [synth.torch_weights_bf16(shapes[l][0], shapes[l][1], synth.seed_for(CFG, l // 7, l % 7), dev)
               for l in range(L)]
        usk.build(plan08, w8_, sk08)
        del w8_
        usk.check(plan08)
        ms08 = time_pass(plan08, sk08)
        pk, pk_s = peaks.get("bf16_tflops", 1666.6), peaks.get("bf16_tflops_sustained", 1352.0)
        c4 = {"workload": "c4: Llama-3.2-1B prefill, 2048 tokens x batch 8 (T = 16384), all 112 linears, M=3",
              "bpw_0.5": {"ms_per_pass": ms05, "ms_per_pass_eager": ms05_eager,
                          "ms_per_pass_per_layer_calls": ms05_single, "TFLOP_per_s": flop / (ms05 * 1e-3) / 1e12,
                          "frac_of_bf16_sustained": flop / (ms05 * 1e-3) / 1e12 / pk_s,
                          "frac_of_bf16_burst": flop / (ms05 * 1e-3) / 1e12 / pk},
              "bpw_0.8": {"ms_per_pass": ms08, "TFLOP_per_s": flop / (ms08 * 1e-3) / 1e12,
                          "frac_of_bf16_sustained": flop / (ms08 * 1e-3) / 1e12 / pk_s,
                          "frac_of_bf16_burst": flop / (ms08 * 1e-3) / 1e12 / pk},
              "flop_per_pass": flop, "calls": "64 usk_linear_batch_tokens per pass (q|k|v, o, gate|up, down of 16 blocks: "
                                                  "one batched reconstruction + one GEMM each, 128 launches) in one CUDA graph "
                                                  "(eager beside; 112 per-layer usk_linear calls beside)",
              "peak_basis": "MEASURED_PEAKS.json bf16 (torch 8192^3): sustained for a 25 ms pass, burst shown beside"}
        del Xp, Yp, Xw, Yw, Yg, ws_p, sk08, plan08
        torch.cuda.empty_cache()

    # ---- BASELINE config 5 at N = 1: Llama-3-8B-shaped linears (224, 6.98 G weights, 13.96 GB bf16)
    #      at 0.5 bpw -- the build of all layers in one call, and the batch-1 decode token as 128
    #      grouped calls in one CUDA graph (the 436 MB sketch exceeds L2: it streams from HBM)
    c5 = None
    if world == 1 and not args.no_8b:
        torch.cuda.empty_cache()
        shapes8 = synth.llama3_8b_shapes()
        L8 = len(shapes8)
        lay8 = args.layout
        try:
            plan8 = usk.plan_allocation(shapes8, bpw=BPW, rows=ROWS, seed=SEED, **LAY)
        except usk.UskError as e:  # 8B gate/up chunks (N = 149) exceed shared memory in the query layout
            if e.status != usk.EUNSUPPORTED:
                raise
            lay8 = "unit_major"
            plan8 = usk.plan_allocation(shapes8, bpw=BPW, rows=ROWS, seed=SEED)
        sk8 = plan8.new_sketch(dev)
        w8 = [synth.torch_weights_bf16(o, i, synth.seed_for(5, l // 7, l % 7), dev) for l, (o, i) in enumerate(shapes8)]
        usk.build(plan8, w8, sk8)
        bt = []
        for _ in range(3):
            flush.fill_(3)
            torch.cuda.synchronize()
            ev0.record()
            usk.build(plan8, w8, sk8)
            ev1.record()
            torch.cuda.synchronize()
            bt.append(ev0.elapsed_time(ev1))
        b8_ms = float(np.median(bt))
        del w8
        torch.cuda.empty_cache()
        usk.check(plan8)
        groups8 = []
        for blk in range(L8 // 7):
            base = 7 * blk
            groups8 += [[base, base + 1, base + 2], [base + 3], [base + 4, base + 5], [base + 6]]
        x8 = [synth.torch_vector(shapes8[g[0]][1], 2000 + gi, dev, torch.bfloat16)[0] for gi, g in enumerate(groups8)]
        y8 = [torch.empty(o, dtype=torch.float32, device=dev) for o, i in shapes8]
        ws8 = [usk.new_batch_workspace(plan8, g, device=dev) for g in groups8]

        def step8():
            for gi, g in enumerate(groups8):
                usk.linear_batch(plan8, sk8, g, x8[gi], [y8[l] for l in g], ws8[gi])

        g8, l8 = capture(step8)
        ms8 = time_steps(g8, step8, max(20, args.steps // 4), args.warmup)
        n8 = sum(o * i for o, i in shapes8)
        c5 = {"workload": "c5 at N=1: Llama-3-8B-shaped 224 linears, 0.5 bpw, M=3",
              "decode_tokens_per_s": 1000.0 / ms8, "decode_ms_per_step": ms8,
              "decode_weights_per_s": n8 * 1000.0 / ms8, "launches_per_step": l8,
              "build_ms": b8_ms, "build_GB_per_s": n8 * (2 + BPW / 8) / (b8_ms * 1e-3) / 1e9,
              "build_hbm_frac": n8 * (2 + BPW / 8) / (b8_ms * 1e-3) / 1e9 / peaks["hbm_gbs"],
              "sketch_MB": plan8.sketch_bytes / 1e6, "weights": n8, "layout": lay8}
        del sk8, plan8, ws8, y8, x8, g8
        torch.cuda.empty_cache()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        getw = host_block0_weights(shapes)
        ncores = max(1, len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count() or 1)
        cpu = oracle_decode_sample(shapes, getw, budget_s=args.cpu_budget, threads=ncores)   # all host cores
        one = oracle_decode_sample(shapes, getw, budget_s=args.cpu_budget / 2, threads=1)
        cpu.pop("weights_per_s", None)
        one.pop("weights_per_s", None)
        one.pop("host", None)
        cpu["single_thread"] = one

    if rank == 0:
        line = {
            "metric": METRIC, "value": tok_s, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (seeded random bf16 weights shaped like Llama-3.2-1B; synth/ recipe)",
            "config": {"workload": "c3: Llama-3.2-1B all 112 linears, batch-1 decode via fused sketch-GEMV",
                       "bpw": BPW, "rows": ROWS, "granularity": "row (1 input dim per unit)", "classes": 1,
                       "sketch_MB": sketch_bytes / 1e6, "weights": numel, "l2": "flushed (256 MB write) before each step",
                       "parallelism": ((f"output-sharded x{world}, one NCCL all-gather per grouped call "
                                        f"({len(groups)} per token, in the graph)") if args.collective == "nccl" else
                                       (f"output-sharded x{world}, y all-gather fused into the reduce kernel "
                                        f"(NVLink peer stores + flags, symmetric memory)")) if world > 1 else "single GPU",
                       "graph": use_graph, "launches_per_step": launches_per_step,
                       "grouping": "q|k|v, o, gate|up, down per block share x (usk_linear_batch)"},
            "per_linear_launches": {"ms_per_step": ms_single, "tokens_per_s": 1000.0 / ms_single,
                                    "launches_per_step": launches_one, "bitwise_equal_to_grouped": same},
            "y_sha256": y_sha,
            "collectives_per_step": len(groups) if world > 1 else 0,
            "weights_reconstructed_per_s": tok_s * numel,
            "reconstruct_standalone": {"weights_per_s": rec_wps, "GB_per_s_written": rec_wps * 2 / 1e9,
                                       "hbm_frac": rec_wps * (2 + 2 * BPW / 16) / 1e9 / peaks["hbm_gbs"]},
            "build": {"ms": build_ms, "replicate_ms": replicate_ms, "weights_per_s": owned_w / (build_ms * 1e-3),
                      "GB_per_s": owned_w * (2 + BPW / 8) / (build_ms * 1e-3) / 1e9},
            "roofline": {"bound": "alu", "achieved": achieved, "peak": gather_floor, "unit": "Gweight/s",
                         "frac": achieved / gather_floor, "traffic": traffic,
                         "kernel": ("k_qgemv (+ k_qreduce)" if QL else "k_gemv_fast (+ k_gemv_reduce)") +
                                   ": the whole timed graph",
                         "peak_basis": (f"shared-memory bandwidth floor (SURVEY 8(d) d.3): M = {ROWS} cell gathers "
                                        f"per weight, " + ("2-B cells, 8 per 16-B load (query layout)" if QL else
                                                           "one 4-B word per lookup") +
                                        f", 128 B/clk/SM -> {per_clk:.2f} weight/clk/SM x {n_sm} SMs x "
                                        f"{f_peak / 1e6:.0f} MHz"),
                         "lds_floor_32bit_words": n_sm * 32.0 / ROWS * f_peak / 1e9,
                         "issue_line": {"peak": alu_peak, "frac": achieved / alu_peak,
                                        "basis": f"{ISSUE:.3f} warp-instructions per 32 weights per SMSP, 1 issue/clk"},
                         "isolated_launch_ms_per_step": sum_kern,
                         "hbm_frac": sketch_bytes / (ms_per_step * 1e-3) / 1e9 / peaks["hbm_gbs"]},
            "e2e": {"value": 1000.0 / e2e_ms, "unit": UNIT, "h2d_bytes_per_step": int(Xh.numel() * 2),
                    "y_to_host": ("reduce kernels store y into pinned host memory (zero-copy)"
                                  if e2e_zc_ms is not None and e2e_zc_ms <= e2e_copy_ms else "cudaMemcpy D2H after the step"),
                    "tokens_per_s_copy_back": 1000.0 / e2e_copy_ms,
                    "tokens_per_s_zero_copy": (1000.0 / e2e_zc_ms) if e2e_zc_ms else None,
                    "d2h_bytes_per_step": int(Yh.numel() * 4)},
            "gpu_launches": int(launches_per_step * args.steps),
            "clocks": clk,
        }
        if cpu is not None:
            line["cpu_baseline"] = cpu
        if q4 is not None:
            line["paper_point_q4"] = q4
        if cls is not None:
            line["importance_classes_rows"] = cls
        if orow is not None:
            line["output_row_units"] = orow
        if p67 is not None:
            line["paper_six_of_seven"] = p67
        if um is not None:
            line["unit_major_usk_x"] = um
        if c5 is not None:
            line["llama3_8b_n1"] = c5
        if c4 is not None:
            line["prefill_c4"] = c4
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


# ----------------------------------------------------------------------------- N > 1 host logic on CPU
def run_dist_selftest(args):
    """The N > 1 path's host logic without GPUs (gloo): output shards per grouped call laid out in
    one buffer and gathered by one collective, the layer-sharded sketch replicated by per-layer
    broadcasts.  Shard outputs and sketch bytes are synthetic functions of (layer, row) / (layer,
    byte), so rank 0's assembled y and sketch must hash the same for every N."""
    import hashlib

    import torch
    import torch.distributed as dist
    from paper_2506_17255_b200 import dist as udist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        dist.init_process_group("gloo")
    shapes = synth.llama32_1b_shapes()
    L = len(shapes)
    groups = []
    for b in range(L // 7):
        base = 7 * b
        groups += [[base, base + 1, base + 2], [base + 3], [base + 4, base + 5], [base + 6]]

    def y_true(l, o0, o1):  # stand-in for a linear's outputs: exact in fp32
        o = torch.arange(o0, o1, dtype=torch.float64)
        return (torch.sin(o * 0.37 + l) * 1000).round().to(torch.float32) / 8

    collectives, ys = 0, []
    for g in groups:
        outs = [shapes[l][0] for l in g]
        lay, pad = udist.group_shard_layout(outs, rank, world)
        buf = torch.zeros(pad, dtype=torch.float32)
        for (o0, o1, off), l in zip(lay, g):
            buf[off:off + o1 - o0] = y_true(l, o0, o1)
        if world > 1:
            full = torch.zeros(world * pad, dtype=torch.float32)
            udist.allgather_group(buf, full)
            collectives += 1
        else:
            full = buf
        ys += udist.assemble_group(full, outs, world)
    Y = torch.cat(ys)
    # layer-sharded build + one-time replication: owners write their layers' regions
    sizes = [o * i // 256 for o, i in shapes]
    offs = np.cumsum([0] + sizes)
    sk = torch.zeros(int(offs[-1]), dtype=torch.uint8)
    for l in udist.owned_layers(L, rank, world):
        n = sizes[l]
        sk[offs[l]:offs[l + 1]] = ((torch.arange(n) * 131 + l * 7) % 251).to(torch.uint8)
    if world > 1:
        udist.replicate_sketch(sk, [(int(offs[l]), int(offs[l + 1])) for l in range(L)], world)
    ok = all(torch.equal(Y[sum(shapes[k][0] for k in range(l)):sum(shapes[k][0] for k in range(l + 1))],
                         y_true(l, 0, shapes[l][0])) for l in range(L))
    if rank == 0:
        print(json.dumps({"selftest": "dist", "n_gpus": world, "y_sha256": hashlib.sha256(Y.numpy().tobytes()).hexdigest(),
                          "sketch_sha256": hashlib.sha256(sk.numpy().tobytes()).hexdigest(), "y_exact": ok,
                          "collectives_per_step": collectives}), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def spawn_ranks(args):
    """`--gpus N` without a launcher: run this script under torch.distributed.run, one rank per GPU
    (127.0.0.1 rendezvous); rank 0 prints the JSON line."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd, cwd=ROOT).returncode


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="usk", choices=["usk", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    ap.add_argument("--ref-step-s", type=float, default=None, help="--impl reference: oracle seconds per step")
    ap.add_argument("--no-q4", action="store_true", help="skip the extra plans (q4 states, classes, output-row units)")
    ap.add_argument("--collective", default="nccl", choices=["nccl", "peer"],
                    help="N > 1 y exchange: one NCCL all-gather per grouped call (default), or the fused peer-store "
                         "epilogue of the reduce kernel over symmetric memory (usk_linear_batch_peers; query layout)")
    ap.add_argument("--layout", default="query", choices=["query", "unit_major"],
                    help="headline plan: query layout + USK-XG keys (default) or the unit-major USK-X plan")
    ap.add_argument("--no-8b", action="store_true", help="skip the Llama-3-8B (config 5) build + decode at N=1")
    ap.add_argument("--no-prefill", action="store_true", help="skip the config-4 prefill passes")
    ap.add_argument("--prefetch-next", action="store_true",
                    help="before each grouped call, usk_prefetch_l2 of the next group's sketch bytes (L2 hint)")
    ap.add_argument("--prefetch", action="store_true",
                    help="start each decode step with usk_prefetch_l2 of the whole sketch (measured: no gain)")
    ap.add_argument("--dist-selftest", action="store_true",
                    help="CPU (gloo) check of the N > 1 launcher and host logic with synthetic shard outputs")
    args = ap.parse_args()
    world_env = os.environ.get("WORLD_SIZE")
    if world_env is None and args.gpus > 1:
        return spawn_ranks(args)
    if world_env is not None and int(world_env) != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but the launcher started WORLD_SIZE={world_env} ranks", file=sys.stderr)
        return 2
    if args.dist_selftest:
        return run_dist_selftest(args)
    if args.impl == "reference":
        return run_reference(args)
    return run_usk(args)


if __name__ == "__main__":
    sys.exit(main())
