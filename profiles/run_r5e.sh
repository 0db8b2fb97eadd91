#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pairing.py tests/test_gpu_stream.py tests/test_gpu_fused_sgd.py -x -q --timeout 240 > gpurun_out/r5e_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r5e_pytest.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/r5e_bench.json 2> gpurun_out/r5e_bench.err
timeout 300 python bench.py --no-cpu-baseline --opt pair_recompute=0 > gpurun_out/r5e_bench_nopair.json 2>> gpurun_out/r5e_bench.err
tail -15 gpurun_out/r5e_pytest.log; cut -c1-700 gpurun_out/r5e_bench.json gpurun_out/r5e_bench_nopair.json; tail -3 gpurun_out/r5e_bench.err
