#!/bin/bash
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_wide -s 20 -c 1 -o gpurun_out/r6k_m1_wide python bench.py --chunks 1 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r6k.log 2>&1
