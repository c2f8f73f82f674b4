# thread-count / registers / subtile sweep (one CTA per SM)
run() { USK_TRACE=1 timeout 300 python tools/trace_step.py --reps 20 > gpurun_out/sw_$1.log 2>&1; echo "== $1"; head -1 gpurun_out/sw_$1.log; grep -A4 "per kind" gpurun_out/sw_$1.log | tail -4; }
b() { USK_NVCC_FLAGS="$1" python paper_2506_17255_b200/build.py > /dev/null 2>&1; }
b "-DUSK_QUERY_THREADS=512 -DUSK_QUERY_MINB=1 -DUSK_SUB_ROWS=16"; run t512_s16
b "-DUSK_QUERY_THREADS=512 -DUSK_QUERY_MINB=1 -DUSK_SUB_ROWS=8"; run t512_s8
b "-DUSK_QUERY_THREADS=768 -DUSK_QUERY_MINB=1 -DUSK_SUB_ROWS=16"; run t768_s16
b "-DUSK_QUERY_THREADS=768 -DUSK_QUERY_MINB=1 -DUSK_SUB_ROWS=8"; run t768_s8
b "-DUSK_QUERY_THREADS=1024 -DUSK_QUERY_MINB=1 -DUSK_SUB_ROWS=16"; run t1024_s16
python paper_2506_17255_b200/build.py --force > /dev/null 2>&1
