#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_order.py tests/test_gpu_pairing.py tests/test_gpu_fused_send.py -x -q --timeout 300 > gpurun_out/r5r_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r5r_pytest.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r5r_bench.json 2> gpurun_out/r5r_bench.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:task_stream_kernel -s 5 -c 1 \
    -o gpurun_out/r5r_streamF python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r5r_ncu_streamF.log 2>&1
tail -3 gpurun_out/r5r_pytest.log; cut -c1-700 gpurun_out/r5r_bench.json; tail -2 gpurun_out/r5r_ncu_streamF.log
