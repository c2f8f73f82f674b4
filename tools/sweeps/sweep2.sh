# occupancy / subtile sweep of the decode step (tools/trace_step.py, USK_TRACE on)
run() { USK_TRACE=1 timeout 300 python tools/trace_step.py --reps 20 > gpurun_out/sw_$1.log 2>&1; echo "== $1"; head -1 gpurun_out/sw_$1.log; grep -A4 "per kind" gpurun_out/sw_$1.log | tail -4; }
python paper_2506_17255_b200/build.py > /dev/null
USK_GEMV_CPS=2 USK_GEMV_SMEM_KB=112 run s8_cps2
USK_GEMV_CPS=2 USK_GEMV_SMEM_KB=112 USK_UPL=2 run s8_cps2_upl2
USK_GEMV_CPS=1 USK_GEMV_SMEM_KB=176 run s8_cps1
USK_NVCC_FLAGS="-DUSK_SUB_ROWS=16" python paper_2506_17255_b200/build.py > /dev/null
USK_GEMV_CPS=2 USK_GEMV_SMEM_KB=112 run s16_cps2
USK_NVCC_FLAGS="-DUSK_QUERY_THREADS=1024 -DUSK_QUERY_MINB=1" python paper_2506_17255_b200/build.py > /dev/null
USK_GEMV_CPS=1 USK_GEMV_SMEM_KB=220 run s8_t1024
python paper_2506_17255_b200/build.py --force > /dev/null
