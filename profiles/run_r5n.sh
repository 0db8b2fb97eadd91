#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ln_dropout.py tests/test_gpu_stream.py -x -q --timeout 300 > gpurun_out/r5n_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r5n_pytest.log
tail -25 gpurun_out/r5n_pytest.log
