USK_NVCC_FLAGS="-DUSK_QUERY_THREADS=512 -DUSK_QUERY_MINB=1 -DUSK_SUB_ROWS=8" python paper_2506_17255_b200/build.py > /dev/null 2>&1
USK_TRACE=1 timeout 300 python tools/trace_step.py --reps 5 --npz gpurun_out/raw_t512.npz > gpurun_out/sw_raw_t512.log 2>&1
head -1 gpurun_out/sw_raw_t512.log
python paper_2506_17255_b200/build.py --force > /dev/null 2>&1
