# ncu --set full of the F task (task_stream_kernel<false,1>) and a paired backward task (<true,2>) at HEAD; phase stamps
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k "regex:ILb0ELi1E" -s 5 -c 1 \
    -o gpurun_out/r7l_streamF python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r7l_ncu_streamF.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k "regex:ILb1ELi2E" -s 5 -c 1 \
    -o gpurun_out/r7l_streamB2 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r7l_ncu_streamB2.log 2>&1
timeout 300 python profiles/st_phases.py blocks=8 > gpurun_out/r7l_phases_fwd.txt 2>&1
tail -2 gpurun_out/r7l_ncu_streamF.log gpurun_out/r7l_ncu_streamB2.log; tail -2 gpurun_out/r7l_phases_fwd.txt
