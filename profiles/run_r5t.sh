#!/bin/bash
# C5 with the tcgen05 attention (default) vs the mma.sync kernels; 4-layer ncu launch list
mkdir -p gpurun_out
timeout 900 python profiles/bench_c5.py > gpurun_out/r5t_c5_tc.json 2> gpurun_out/r5t_c5_tc.err
TGP_ATTN_TC=0 timeout 900 python profiles/bench_c5.py > gpurun_out/r5t_c5_mma.json 2> gpurun_out/r5t_c5_mma.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
    --log-file gpurun_out/r5t_c5_launches_4layers.csv python profiles/bench_c5.py --layers 4 --seqs 8 --chunks 8 --steps 1 --warmup 1 > /dev/null 2>&1
TGP_ATTN_TC=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
    --log-file gpurun_out/r5t_c5_launches_4layers_mma.csv python profiles/bench_c5.py --layers 4 --seqs 8 --chunks 8 --steps 1 --warmup 1 > /dev/null 2>&1
cut -c1-500 gpurun_out/r5t_c5_tc.json gpurun_out/r5t_c5_mma.json; tail -2 gpurun_out/r5t_c5_tc.err
