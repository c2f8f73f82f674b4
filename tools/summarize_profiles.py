"""Write the committed profiles/ summaries from a tools/profile_round.sh run (gpurun_out/).

  python tools/summarize_profiles.py [--tag r1]

Produces:
  profiles/<tag>_bench.jsonl          bench.py line (appended) + the --impl reference line
  profiles/<tag>_launches_bench.txt   ncu launch list of the bench command, per kernel
  profiles/<tag>_ncu_full_summary.txt per-launch key metrics of the `ncu --set full` capture
  profiles/<tag>_decode_trace.txt     in-graph per-launch timeline of one decode step
  profiles/traffic.json               DRAM bytes per k_gemv_fast launch vs algorithmic
"""
import argparse
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
sys.path.insert(0, ROOT)
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

ap = argparse.ArgumentParser()
ap.add_argument("--tag", default="r1")
args = ap.parse_args()


def json_line(path):
    for line in reversed(open(path).read().splitlines()):
        if line.startswith("{"):
            return line
    return None


# ---- bench lines
bl = json_line(os.path.join(OUT, "bench_full.log"))
rl = json_line(os.path.join(OUT, "bench_ref.log")) if os.path.exists(os.path.join(OUT, "bench_ref.log")) else None
bp = os.path.join(PROF, f"{args.tag}_bench.jsonl")
have = open(bp).read().splitlines() if os.path.exists(bp) else []
with open(bp, "a") as f:
    for line in (bl, rl):
        if line and line not in have:
            f.write(line + "\n")

# ---- launch list
import launches  # noqa: E402

d = launches.summarise(os.path.join(OUT, "launches_bench.csv"))
tot = sum(sum(v) for v in d.values())
with open(os.path.join(PROF, f"{args.tag}_launches_bench.txt"), "w") as f:
    f.write("# ncu --metrics gpu__time_duration.sum --clock-control none of `python bench.py --steps 3 --warmup 3 "
            "--no-cpu-baseline` (whole process: plans, builds, warm-up + timed decode graphs, per-linear graphs,\n"
            "# isolated per-call timing, 112 reconstructs, e2e, then the extra plans: q4 states, importance classes\n"
            "# with per-class rows, output-row units, Llama-3-8B at N=1).  Per-launch times are cold-cache and\n"
            "# serialised by ncu; the shares, not the absolutes, compare with the bench.\n")
    f.write(f"{'kernel':36s} {'n':>5s} {'mean_us':>10s} {'total_us':>11s} {'share':>6s}\n")
    for k, v in d.items():
        f.write(f"{k:36s} {len(v):5d} {sum(v) / len(v):10.2f} {sum(v):11.2f} {sum(v) / tot:6.1%}\n")

# ---- ncu full summary
rep = os.path.join(OUT, "prof_round.ncu-rep")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr = rows[0]
keys = ["gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "smsp__inst_executed.sum"]
gemv_bytes = []
with open(os.path.join(PROF, f"{args.tag}_ncu_full_summary.txt"), "w") as f:
    f.write("# ncu --set full --clock-control none --import-source on of tools/prof_kernels.py --reps 1 --prefill\n"
            "# order: per grouped call (q|k|v, o, gate|up, down of Llama-3.2-1B block 0, 0.5 bpw, M=3) the compute\n"
            "# kernel (k_qgemv on the query layout, k_gemv_fast unit-major) + its reduce; the block build; the gate\n"
            "# reconstruct; the 2048-token gate|up prefill (one batched reconstruction + one tcgen05 GEMM).\n"
            "# Serialised, cold-cache replays (ncu), not bench numbers.\n")
    for row in rows[2:]:
        r = dict(zip(hdr, row))
        name = r.get("Kernel Name", "")
        rec = {"kernel": name[:70]}
        for k in keys:
            if k in r:
                rec[k] = r[k]
        f.write(json.dumps(rec) + "\n")
        if "k_gemv_fast" in name or "k_qgemv" in name:
            unit = r.get("dram__bytes_read.sum", "0")
            gemv_bytes.append((float(r["dram__bytes_read.sum"]) + float(r["dram__bytes_write.sum"])) * 1e6)

# ---- traffic.json: DRAM bytes per decode-kernel launch (MB in the raw page) vs algorithmic
if gemv_bytes:
    # algorithmic bytes of the 4 grouped calls of block 0 (USK-XG query plan, the bench's): the block's
    # sketch bytes + x (bf16) + the fp32 chunk partials [rows][in / 256]
    import oracle  # noqa: E402  (CPU plan: same cell counts as the GPU plan, tests/test_gpu_query_layout)
    import synth  # noqa: E402
    shapes = synth.llama_block(2048, 512, 8192)
    cells = oracle.plan(shapes, 0.5, M=3, dtype=oracle.BF16, seed=0x5EED000000000003,
                        hash_kind=oracle.HASH_XG).total_cells
    xy = 2 * (2048 + 2048 + 2048 + 8192) + sum(4 * o * (i // 256) for o, i in shapes)
    alg = (2 * cells + xy) / len(gemv_bytes)
    tp = os.path.join(PROF, "traffic.json")
    tj = json.load(open(tp)) if os.path.exists(tp) else {}
    tj.update({"k_qgemv_bytes_per_launch": sum(gemv_bytes) / len(gemv_bytes),
               "k_qgemv_algorithmic_bytes_per_launch": alg,
               "k_qgemv_source": "ncu --set full dram__bytes_read.sum + dram__bytes_write.sum of the %d grouped k_qgemv "
                                 "launches of Llama-3.2-1B block 0 (profiles/%s_ncu_full_summary.txt), averaged per "
                                 "launch; algorithmic = the block's query-layout sketch bytes + x (bf16) + fp32 chunk "
                                 "partials over the same launches" % (len(gemv_bytes), args.tag)})
    json.dump(tj, open(tp, "w"), indent=1)

# ---- decode trace
tl = os.path.join(OUT, "trace_round.log")
if os.path.exists(tl):
    with open(os.path.join(PROF, f"{args.tag}_decode_trace.txt"), "w") as f:
        f.write("# USK_TRACE=1 tools/trace_step.py --reps 30: one decode step (Llama-3.2-1B, 64 grouped calls = "
                "128 launches in one CUDA graph, L2 flushed), per-launch %globaltimer spans (us).\n"
                "# stage = CTA start -> chunk staged + griddepcontrol.wait passed; comp = -> last subtile; "
                "gap < 0 = overlap with the previous launch (PDL).\n")
        f.write(open(tl).read())
print("profiles written")
