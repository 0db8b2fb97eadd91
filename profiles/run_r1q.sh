OUT=gpurun_out; mkdir -p $OUT
timeout 300 python -m pytest tests/test_gpu_stream.py -x -q --timeout 120 > $OUT/pytest_stream_r1q.log 2>&1; echo "rc=$?" >> $OUT/pytest_stream_r1q.log
tail -15 $OUT/pytest_stream_r1q.log
for v in 0 1; do timeout 120 python profiles/st_phases.py blocks=32 variant=$v | tail -1 | sed "s/^/variant $v: /" >> $OUT/st_var_r1q.txt 2>&1; done
timeout 120 python profiles/st_phases.py blocks=4 >> $OUT/st_var_r1q.txt 2>&1
cat $OUT/st_var_r1q.txt
