#!/bin/bash
# Evidence run for profiles/: bench line, ncu launch list of the same bench command, one
# `ncu --set full` capture of the top kernel (the grouped gate|up sketch-GEMV), clocks.
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv -lms 200 > gpurun_out/clocks.csv &
SMI=$!
python bench.py --steps 30 --warmup 5 > gpurun_out/bench_full.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_full.log
kill $SMI
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "launches rc=$?" >> gpurun_out/ncu_launch.log
python tools/prof_kernels.py --reps 1 > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_query_fast|k_build_fast|k_gemm_tc" -s 1 -c 8 -o gpurun_out/prof_round python tools/prof_kernels.py --reps 1 --prefill > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?" >> gpurun_out/ncu_full.log
