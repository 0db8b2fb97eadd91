#!/bin/bash
mkdir -p gpurun_out
for a in "f 1" "fb 1"; do timeout 120 python profiles/diag/determinism.py 4096 2 64 4 $a 2>&1 | tail -1; done > gpurun_out/r5u_det.txt 2>&1
timeout 300 python profiles/st_time.py 32 > gpurun_out/r5u_st_time.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_stream.py tests/test_gpu_pairing.py tests/test_gpu_fused_send.py tests/test_gpu_fused_sgd.py -x -q --timeout 300 > gpurun_out/r5u_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r5u_pytest.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r5u_bench.json 2> gpurun_out/r5u_bench.err
timeout 300 python profiles/st_phases.py blocks=8 > gpurun_out/r5u_phases_fwd.txt 2>&1
cat gpurun_out/r5u_det.txt gpurun_out/r5u_st_time.txt; tail -3 gpurun_out/r5u_pytest.log; cut -c1-500 gpurun_out/r5u_bench.json; tail -2 gpurun_out/r5u_phases_fwd.txt
