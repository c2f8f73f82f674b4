python paper_2506_17255_b200/build.py > /dev/null 2>&1
timeout 300 python tools/prof_kernels.py > gpurun_out/pk.log 2>&1 && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_gemv_fast -c 4 -o gpurun_out/prof_gemv2 -f python tools/prof_kernels.py > gpurun_out/ncu_gemv2.log 2>&1
tail -3 gpurun_out/ncu_gemv2.log
