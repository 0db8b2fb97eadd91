OUT=gpurun_out; mkdir -p $OUT
timeout 300 python -m pytest tests/test_gpu_stream.py -x -q --timeout 120 2>&1 | tail -5
for v in 0 1; do timeout 120 python profiles/st_phases.py blocks=32 variant=$v | tail -1 | sed "s/^/fwd variant $v: /"; done
timeout 120 python profiles/st_phases.py blocks=32 bwd=1 | tail -1 | sed "s/^/bwd: /"
timeout 120 python profiles/st_phases.py blocks=4 2>&1
timeout 120 python profiles/step_breakdown.py 2>&1
