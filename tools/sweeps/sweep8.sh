run() { USK_TRACE=1 timeout 300 python tools/trace_step.py --reps 30 > gpurun_out/sw_$1.log 2>&1; echo "== $1 $(head -1 gpurun_out/sw_$1.log)"; }
python paper_2506_17255_b200/build.py > /dev/null 2>&1
run s16_220
USK_SWITCH_ITEMS=12 run s16_220_p12
USK_SWITCH_ITEMS=30 run s16_220_p30
USK_GEMV_SMEM_KB=192 run s16_192
