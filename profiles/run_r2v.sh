for v in 0 8192 0 8192; do timeout 60 python profiles/step_breakdown.py test_stream_variant=$v 2>&1 | head -4; done
