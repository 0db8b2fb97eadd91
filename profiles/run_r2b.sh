timeout 300 python -m pytest tests/test_gpu_stream.py -x -q --timeout 120 2>&1 | tail -5
timeout 120 python profiles/st_time.py 0 1
timeout 120 python profiles/st_phases.py blocks=32 bwd=1 | tail -1 | sed "s/^/bwd: /"
timeout 120 python profiles/st_phases.py blocks=4 bwd=1 2>&1 | head -7
timeout 120 python profiles/step_breakdown.py 2>&1
