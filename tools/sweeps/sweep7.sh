run() { USK_TRACE=1 timeout 300 python tools/trace_step.py --reps 30 > gpurun_out/sw_$1.log 2>&1; echo "== $1 $(head -1 gpurun_out/sw_$1.log)"; }
python paper_2506_17255_b200/build.py > /dev/null 2>&1
run base
USK_SWITCH_ITEMS=0 run p0
USK_SWITCH_ITEMS=20 run p20
USK_SWITCH_ITEMS=60 run p60
USK_GEMV_SMEM_KB=220 run smem220
USK_GEMV_SMEM_KB=170 run smem170
USK_NVCC_FLAGS="-DUSK_SUB_ROWS=16" python paper_2506_17255_b200/build.py > /dev/null 2>&1
run sub16
USK_NVCC_FLAGS="-DUSK_GEMV_MAXREG=96" python paper_2506_17255_b200/build.py > /dev/null 2>&1
run reg96
python paper_2506_17255_b200/build.py --force > /dev/null 2>&1
