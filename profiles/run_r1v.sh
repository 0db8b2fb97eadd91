OUT=gpurun_out; mkdir -p $OUT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:task_stream_kernel -s 2 -c 1 -o $OUT/prof_stream_r1v python profiles/st_phases.py blocks=8 > $OUT/ncu_stream_r1v.log 2>&1
tail -2 $OUT/ncu_stream_r1v.log
