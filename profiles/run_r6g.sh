#!/bin/bash
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 40 -c 1 -o gpurun_out/r6g_m4_gemm python bench.py --chunks 4 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r6g_m4_full.log 2>&1
