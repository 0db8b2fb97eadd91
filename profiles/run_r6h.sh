#!/bin/bash
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r6h_m4_launches.csv python bench.py --chunks 4 --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/r6h_m4.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r6h_m8_launches.csv python bench.py --chunks 8 --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/r6h_m8.log 2>&1
