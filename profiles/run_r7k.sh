# HEAD measurement set: sanitizers (incl. async ABI), ncu launch list, ncu --set full of the F task and a
# paired backward task, C3 sweep, full C5
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck racecheck; do
  timeout 900 $CS --tool $tool --print-limit 20 --log-file gpurun_out/r7k_san_$tool.log python profiles/diag/sanitize_case.py 0 4 > gpurun_out/r7k_san_${tool}_stdout.log 2>&1
  echo "rc=$?" >> gpurun_out/r7k_san_${tool}_stdout.log
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
    --log-file gpurun_out/r7k_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:task_stream_kernel<0, 1>" -s 5 -c 1 \
    -o gpurun_out/r7k_streamF python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r7k_ncu_streamF.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:task_stream_kernel<1, 2>" -s 5 -c 1 \
    -o gpurun_out/r7k_streamB2 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r7k_ncu_streamB2.log 2>&1
for m in 32 8 4 1; do for ck in except_last always never; do
  timeout 300 python bench.py --chunks $m --checkpoint $ck --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r7k_c3_${m}_${ck}.json 2>/dev/null
  python -c "
import json
d=json.load(open('gpurun_out/r7k_c3_${m}_${ck}.json'))
t=d['pipeline']['tasks']
print(f\"m={d['config']['chunks']:3d} {d['config']['checkpoint']:12s} {d['ms_per_step']:8.2f} ms/step {d['value']:8.0f} samples/s  F {t.get('F',{}).get('median_us',0):7.0f} us  F' {t.get(\\\"F'\\\",{}).get('median_us',0):7.0f} us  B {t.get('B',{}).get('median_us',0):7.0f} us  W {t.get('W',{}).get('median_us',0):7.0f} us  dominant {d['roofline']['kernel'][:22]} frac {d['roofline']['frac']:.3f}\")
" >> gpurun_out/r7k_c3_sweep.txt 2>&1
done; done
timeout 900 python profiles/bench_c5.py --layers 48 --steps 2 --warmup 1 > gpurun_out/r7k_c5.json 2> gpurun_out/r7k_c5.err
cat gpurun_out/r7k_c3_sweep.txt; tail -1 gpurun_out/r7k_c5.json | cut -c1-400
for t in memcheck synccheck racecheck; do echo "== $t"; tail -3 gpurun_out/r7k_san_$t.log; tail -4 gpurun_out/r7k_san_${t}_stdout.log; done
