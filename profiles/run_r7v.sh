# C5 4-layer launch list at HEAD (8 sequences, m = 8) for the per-kernel share
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
    --log-file gpurun_out/r7v_c5_launches.csv python profiles/bench_c5.py --layers 4 --seqs 8 --chunks 8 --steps 1 --warmup 1 > gpurun_out/r7v_c5.log 2>&1
timeout 600 python profiles/bench_c5.py --layers 8 --seqs 8 --chunks 8 --steps 3 --warmup 2 > gpurun_out/r7v_c5_8l.json 2>&1
tail -1 gpurun_out/r7v_c5_8l.json | cut -c1-300
