#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_fused_sgd.py -x -q --timeout 300 > gpurun_out/r5d_pytest.log 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r5d_bench.json 2> gpurun_out/r5d_bench.err
timeout 600 python bench.py --no-cpu-baseline --unfused-sgd > gpurun_out/r5d_bench_unfused.json 2>> gpurun_out/r5d_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv \
    --log-file gpurun_out/r5d_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
tail -5 gpurun_out/r5d_pytest.log; cat gpurun_out/r5d_bench.json gpurun_out/r5d_bench_unfused.json | cut -c1-600; tail -3 gpurun_out/r5d_bench.err
