timeout 300 python -m pytest tests/test_gpu_stream.py tests/test_gpu_multiproc.py -x -q --timeout 200 2>&1 | tail -3
timeout 120 python profiles/st_time.py 0 1
timeout 120 python profiles/step_breakdown.py 2>&1
