#!/bin/bash
mkdir -p gpurun_out
timeout 200 python profiles/diag/determinism.py 4096 2 64 4 f 1 > gpurun_out/r6a_det_f.txt 2>&1; tail -3 gpurun_out/r6a_det_f.txt
timeout 200 python profiles/diag/determinism.py 4096 2 64 4 fb 1 > gpurun_out/r6a_det_fb.txt 2>&1; tail -3 gpurun_out/r6a_det_fb.txt
timeout 200 python profiles/st_time.py 32 > gpurun_out/r6a_st.txt 2>&1; tail -3 gpurun_out/r6a_st.txt
timeout 900 python -m pytest -x -q tests/test_gpu_stream.py tests/test_gpu_pairing.py tests/test_gpu_fused_send.py tests/test_gpu_fused_sgd.py > gpurun_out/r6a_tests.txt 2>&1; tail -5 gpurun_out/r6a_tests.txt
timeout 300 python bench.py > gpurun_out/r6a_bench.txt 2>&1; tail -1 gpurun_out/r6a_bench.txt | cut -c1-600
