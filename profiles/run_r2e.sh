timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 2>&1 | tail -3
timeout 120 python profiles/step_breakdown.py 2>&1
timeout 120 python profiles/step_breakdown.py dw_persistent=0 2>&1 | head -1
