set -x
run() { USK_TRACE=1 timeout 300 python tools/trace_step.py --reps 20 > gpurun_out/sw_$1.log 2>&1; tail -6 gpurun_out/sw_$1.log | head -1; grep -A4 "per kind" gpurun_out/sw_$1.log; head -1 gpurun_out/sw_$1.log; }
USK_GEMV_CPS=2 USK_GEMV_SMEM_KB=112 run cps2_112
USK_GEMV_CPS=2 USK_GEMV_SMEM_KB=112 USK_UPL=2 run cps2_112_upl2
USK_GEMV_CPS=1 USK_GEMV_SMEM_KB=176 run cps1_176
USK_NVCC_FLAGS="-DUSK_QUERY_THREADS=1024 -DUSK_QUERY_MINB=1" python paper_2506_17255_b200/build.py > gpurun_out/build1024.log 2>&1
USK_GEMV_CPS=1 USK_GEMV_SMEM_KB=220 run t1024_220
USK_GEMV_CPS=1 USK_GEMV_SMEM_KB=220 USK_UPL=2 run t1024_220_upl2
