timeout 200 python -m pytest tests/test_gpu_stream.py -x -q --timeout 60 2>&1 | tail -2
timeout 60 python profiles/st_time.py 0 8192 0 8192
timeout 60 python profiles/step_breakdown.py 2>&1
