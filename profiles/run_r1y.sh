OUT=gpurun_out; mkdir -p $OUT
timeout 300 python -m pytest tests/test_gpu_stream.py tests/test_gpu_gemm.py -x -q --timeout 120 2>&1 | tail -5
timeout 120 python profiles/step_breakdown.py 2>&1
