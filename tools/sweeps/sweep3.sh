python paper_2506_17255_b200/build.py > /dev/null
USK_GEMV_CPS=2 USK_GEMV_SMEM_KB=112 USK_TRACE=1 timeout 300 python tools/trace_step.py --reps 5 --npz gpurun_out/raw_cps2.npz > gpurun_out/sw_raw_cps2.log 2>&1
head -1 gpurun_out/sw_raw_cps2.log
