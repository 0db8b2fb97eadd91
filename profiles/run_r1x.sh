OUT=gpurun_out; mkdir -p $OUT
for v in 1 1025 3 1027; do timeout 120 python profiles/st_phases.py blocks=32 variant=$v | tail -1 | sed "s/^/fwd variant $v: /" >> $OUT/st_var_r1x.txt 2>&1; done
cat $OUT/st_var_r1x.txt
