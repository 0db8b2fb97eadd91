OUT=gpurun_out; mkdir -p $OUT
(timeout 120 python profiles/st_phases.py blocks=4; timeout 120 python profiles/st_phases.py blocks=4 nodep=1; timeout 120 python profiles/st_phases.py blocks=4 bwd=1; timeout 120 python profiles/st_phases.py blocks=32 nodep=1 | tail -3 ; timeout 120 python profiles/st_phases.py blocks=32 | tail -3) > $OUT/st_phases_r1l.txt 2>&1
cat $OUT/st_phases_r1l.txt
