#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/r5k_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r5k_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r5k_smoke.log 2>&1
tail -15 gpurun_out/r5k_pytest_gpu.log; tail -2 gpurun_out/r5k_smoke.log
