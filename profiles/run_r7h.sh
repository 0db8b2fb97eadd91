# paired (F' beside B on half grids) vs unpaired full-grid tasks, after the full-grid copy throttle
mkdir -p gpurun_out
for v in pair nopair pair nopair; do
  if [ $v = pair ]; then O=""; else O="--opt pair_recompute=0"; fi
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline $O > gpurun_out/r7h_bench_$v.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/r7h_bench_$v.json')); t=d['pipeline']['tasks']
print('$v', round(d['ms_per_step'],2), {k: round(v['median_us'],1) for k, v in t.items()}, 'frac', round(d['roofline']['frac'],4))" >> gpurun_out/r7h_summary.txt
done
cat gpurun_out/r7h_summary.txt
