# accumulators sized by row count at the top of TMEM (forward half grid: 14 -> 15 weight slots)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stream.py tests/test_gpu_pairing.py tests/test_gpu_fused_send.py -x -q > gpurun_out/r7n_pytest.txt 2>&1
echo "rc=$?" >> gpurun_out/r7n_pytest.txt
for v in pair nopair pair; do
  if [ $v = pair ]; then O=""; else O="--opt pair_recompute=0"; fi
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline $O > gpurun_out/r7n_bench_$v.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/r7n_bench_$v.json')); t=d['pipeline']['tasks']
print('$v', round(d['ms_per_step'],2), {k: round(v['median_us'],1) for k, v in t.items()}, 'frac', round(d['roofline']['frac'],4))" >> gpurun_out/r7n_summary.txt
done
cat gpurun_out/r7n_summary.txt; tail -n 2 gpurun_out/r7n_pytest.txt
