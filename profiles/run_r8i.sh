# stream-kernel F of a checkpointed micro-batch skips its dead intermediates (option dead_stash): tests + bench A/B
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r8i_pytest_gpu.txt 2>&1
echo "rc=$?" >> gpurun_out/r8i_pytest_gpu.txt
tail -n 2 gpurun_out/r8i_pytest_gpu.txt
for v in on off on off; do
  if [ $v = on ]; then O=""; else O="--opt dead_stash=0"; fi
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline $O > gpurun_out/r8i_bench_$v.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/r8i_bench_$v.json')); t=d['pipeline']['tasks']
print('dead_stash $v', round(d['ms_per_step'],2), {k: round(v['median_us'],1) for k, v in t.items()}, 'frac', round(d['roofline']['frac'],4))" >> gpurun_out/r8i_summary.txt
done
cat gpurun_out/r8i_summary.txt
