OUT=gpurun_out; mkdir -p $OUT
timeout 300 python -m pytest tests/test_gpu_stream.py -x -q --timeout 120 > $OUT/pytest_stream_r1o.log 2>&1; echo "rc=$?" >> $OUT/pytest_stream_r1o.log
tail -3 $OUT/pytest_stream_r1o.log
# pf distance: default 16, none (63<<4=1008), 8 (128), 32 (512), 48 (768)
for v in 0 1008 128 512 768 1; do timeout 120 python profiles/st_phases.py blocks=32 variant=$v | tail -1 | sed "s/^/variant $v: /" >> $OUT/st_var_r1o.txt 2>&1; done
for v in 0 1008 512; do timeout 120 python profiles/st_phases.py blocks=32 bwd=1 variant=$v | tail -1 | sed "s/^/bwd variant $v: /" >> $OUT/st_var_r1o.txt 2>&1; done
timeout 120 python profiles/st_phases.py blocks=4 >> $OUT/st_var_r1o.txt 2>&1
cat $OUT/st_var_r1o.txt
