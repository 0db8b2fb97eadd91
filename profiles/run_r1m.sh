OUT=gpurun_out; mkdir -p $OUT
for v in 1 3 5 9 0 4 8; do timeout 120 python profiles/st_phases.py blocks=32 variant=$v | tail -1 | sed "s/^/variant $v: /" >> $OUT/st_var_r1m.txt 2>&1; done
for v in 0 4; do timeout 120 python profiles/st_phases.py blocks=32 bwd=1 variant=$v | tail -1 | sed "s/^/bwd variant $v: /" >> $OUT/st_var_r1m.txt 2>&1; done
cat $OUT/st_var_r1m.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:task_stream_kernel -s 2 -c 1 -o $OUT/prof_stream_r1m python profiles/st_phases.py blocks=4 > $OUT/ncu_stream_r1m.log 2>&1
tail -3 $OUT/ncu_stream_r1m.log
