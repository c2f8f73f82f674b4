run() { USK_TRACE=1 timeout 300 python tools/trace_step.py --reps 20 > gpurun_out/sw_$1.log 2>&1; echo "== $1"; head -1 gpurun_out/sw_$1.log; grep -A4 "per kind" gpurun_out/sw_$1.log | tail -4; }
python paper_2506_17255_b200/build.py > /dev/null
timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
run t1024
USK_UPL=2 run t1024_upl2
timeout 300 python bench.py --steps 100 --no-cpu-baseline > gpurun_out/bench_j.log 2>&1; tail -c 400 gpurun_out/bench_j.log
