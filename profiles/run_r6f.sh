#!/bin/bash
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 40 -c 1 -o gpurun_out/r6f_m4_gemm python bench.py --chunks 4 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r6f_m4_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 40 -c 1 -o gpurun_out/r6f_m8_gemm python bench.py --chunks 8 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r6f_m8_full.log 2>&1
(export TGP_LIB=$PWD/variants/timing/libtgp.so
for pf in 0 1; do CHUNKS=4 PF=$pf timeout 300 python profiles/gemm_timeline.py 4 2>&1 | head -6; done)
