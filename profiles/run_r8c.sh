# F'/B pairing for per-layer partitions: GPU tests, C3 m = 4 / 8 (except_last, always) and C5 8 layers, pair on / off
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r8c_pytest_gpu.txt 2>&1
echo "rc=$?" >> gpurun_out/r8c_pytest_gpu.txt
tail -n 3 gpurun_out/r8c_pytest_gpu.txt
for v in pair nopair; do
  if [ $v = pair ]; then O=""; else O="--opt pair_recompute=0"; fi
  for m in 4 8; do for ck in except_last always; do
    timeout 300 python bench.py --chunks $m --checkpoint $ck --steps 5 --warmup 3 --no-cpu-baseline $O > gpurun_out/r8c_bench_${v}_${m}_$ck.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/r8c_bench_${v}_${m}_$ck.json')); t=d['pipeline']['tasks']
print('$v m=$m $ck', round(d['ms_per_step'],2), {k: round(v['median_us'],1) for k, v in t.items()})" >> gpurun_out/r8c_summary.txt
  done; done
done
cat gpurun_out/r8c_summary.txt
