OUT=gpurun_out; mkdir -p $OUT
timeout 120 python profiles/st_phases.py blocks=4 > $OUT/st_r1u.txt 2>&1
timeout 120 python profiles/st_phases.py blocks=4 bwd=1 >> $OUT/st_r1u.txt 2>&1
cat $OUT/st_r1u.txt
timeout 300 python -m pytest tests/test_gpu_stream.py -x -q --timeout 120 2>&1 | tail -2
timeout 120 python profiles/step_breakdown.py 2>&1
