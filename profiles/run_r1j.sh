OUT=gpurun_out; mkdir -p $OUT
for o in "persistent=0" "persistent=1" "ckpt=never persistent=0" "ckpt=never persistent=1"; do timeout 300 python profiles/step_breakdown.py $o >> $OUT/breakdown_r1j.txt 2>&1; done
timeout 600 python profiles/modes_bitwise_full.py > $OUT/modes_r1j.txt 2>&1
timeout 300 python profiles/modes_bitwise_full.py persistent=1 >> $OUT/modes_r1j.txt 2>&1
timeout 300 python profiles/pt_phases.py 4 > $OUT/pt_phases_r1j.txt 2>&1
cat $OUT/breakdown_r1j.txt $OUT/modes_r1j.txt $OUT/pt_phases_r1j.txt
