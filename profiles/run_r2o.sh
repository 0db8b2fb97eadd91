timeout 60 python -m pytest tests/test_gpu_stream.py -x -q --timeout 30 -k "full_c2 or ragged" 2>&1 | tail -3
timeout 60 python profiles/st_time.py 0 2048 1 2049
timeout 60 python profiles/step_breakdown.py 2>&1
