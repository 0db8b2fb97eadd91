#!/bin/bash
mkdir -p gpurun_out
export TGP_LIB=$PWD/variants/sk_6/libtgp.so
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r6c_m4_launches.csv python bench.py --chunks 4 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r6c_m4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 40 -c 1 -o gpurun_out/r6c_m4_gemm python bench.py --chunks 4 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r6c_m4_full.log 2>&1
ls -la gpurun_out
