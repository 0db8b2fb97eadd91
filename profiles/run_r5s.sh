#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_gpt2.py -x -q --timeout 600 > gpurun_out/r5s_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r5s_pytest.log
tail -30 gpurun_out/r5s_pytest.log
