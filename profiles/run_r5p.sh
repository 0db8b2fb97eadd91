#!/bin/bash
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/r5p_bench.json 2> gpurun_out/r5p_bench.err
timeout 300 python profiles/st_phases.py blocks=8 > gpurun_out/r5p_phases_fwd.txt 2>&1
for v in ws2_8 ws3_7 ws2_6; do TGP_LIB=variants/libtgp_$v.so timeout 300 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/r5p_bench_$v.json 2>/dev/null; done
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:task_stream_kernel<0, 1>" -s 5 -c 1 \
    -o gpurun_out/r5p_streamF python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r5p_ncu_streamF.log 2>&1
cut -c1-400 gpurun_out/r5p_bench.json; tail -3 gpurun_out/r5p_phases_fwd.txt
for v in ws2_8 ws3_7 ws2_6; do python -c "import json;d=json.load(open('gpurun_out/r5p_bench_$v.json'));print('$v', d['ms_per_step'], d['pipeline']['tasks']['W'])"; done
tail -3 gpurun_out/r5p_ncu_streamF.log
