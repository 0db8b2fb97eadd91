# HEAD (ld.acquire counters): phase stamps, poll back-off sweep, ncu launch list + full capture of the F task
mkdir -p gpurun_out
timeout 300 python profiles/st_phases.py blocks=8 > gpurun_out/r7d_phases_fwd.txt 2>&1
timeout 300 python profiles/st_phases.py blocks=8 bwd=1 > gpurun_out/r7d_phases_bwd.txt 2>&1
for p in 0 16 64 128; do
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --opt stream_poll_ns=$p > gpurun_out/r7d_bench_poll$p.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/r7d_bench_poll$p.json')); t=d['pipeline']['tasks']
print('poll_ns=$p', round(d['ms_per_step'],2), 'F', t['F']['median_us'], 'Fp', t[\"F'\"]['median_us'], 'B', t['B']['median_us'], 'frac', round(d['roofline']['frac'],4))" >> gpurun_out/r7d_poll_sweep.txt
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
    --log-file gpurun_out/r7d_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:task_stream_kernel -s 5 -c 1 \
    -o gpurun_out/r7d_streamF python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r7d_ncu_streamF.log 2>&1
cat gpurun_out/r7d_poll_sweep.txt; tail -3 gpurun_out/r7d_phases_fwd.txt gpurun_out/r7d_phases_bwd.txt
