# per-layer F of a checkpointed micro-batch skips the pre-activation stores too: suite + C5 8 layers + C3 m = 4 / 8 A/B
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r8j_pytest_gpu.txt 2>&1
echo "rc=$?" >> gpurun_out/r8j_pytest_gpu.txt
tail -n 2 gpurun_out/r8j_pytest_gpu.txt
for v in on off on off; do
  if [ $v = on ]; then O=""; else O="--opt dead_stash=0"; fi
  for m in 4 8; do
    timeout 300 python bench.py --chunks $m --checkpoint always --steps 5 --warmup 3 --no-cpu-baseline $O > gpurun_out/r8j_bench_${v}_$m.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/r8j_bench_${v}_$m.json')); t=d['pipeline']['tasks']
print('dead_stash $v m=$m always', round(d['ms_per_step'],2), {k: round(v['median_us'],1) for k, v in t.items()})" >> gpurun_out/r8j_summary.txt
  done
done
cat gpurun_out/r8j_summary.txt
