OUT=gpurun_out; mkdir -p $OUT
for v in 0 2 1 3; do timeout 120 python profiles/st_phases.py blocks=32 variant=$v | tail -1 | sed "s/^/fwd variant $v: /" >> $OUT/st_var_r1w.txt 2>&1; done
for v in 0 2; do timeout 120 python profiles/st_phases.py blocks=32 bwd=1 variant=$v | tail -1 | sed "s/^/bwd variant $v: /" >> $OUT/st_var_r1w.txt 2>&1; done
cat $OUT/st_var_r1w.txt
