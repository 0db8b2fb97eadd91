#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_fused_send.py tests/test_gpu_order.py tests/test_gpu_multiproc.py tests/test_gpu_transport.py tests/test_gpu_pairing.py tests/test_gpu_parity.py -x -q --timeout 300 > gpurun_out/r5l_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r5l_pytest.log
tail -25 gpurun_out/r5l_pytest.log
