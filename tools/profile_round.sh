#!/bin/bash
# Evidence run for profiles/: GPU tests, bench line (clocks sampled), ncu launch list of the same
# bench command, one `ncu --set full` capture of the hot kernels, the in-graph decode trace.
set -u
mkdir -p gpurun_out
python paper_2506_17255_b200/build.py > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
python bench.py > gpurun_out/bench_full.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_full.log
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "launches rc=$?" >> gpurun_out/ncu_launch.log
python tools/prof_kernels.py --reps 1 --prefill > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_qgemv|k_qreduce|k_build_fast|k_qrecon|k_gemm_tc" -c 14 -o gpurun_out/prof_round -f python tools/prof_kernels.py --reps 1 --prefill > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?" >> gpurun_out/ncu_full.log
USK_TRACE=1 python tools/trace_step.py --reps 30 --csv gpurun_out/trace_round.csv > gpurun_out/trace_round.log 2>&1
tail -2 gpurun_out/pytest_gpu.log; tail -c 300 gpurun_out/bench_full.log; tail -1 gpurun_out/ncu_launch.log; tail -1 gpurun_out/ncu_full.log; head -1 gpurun_out/trace_round.log
