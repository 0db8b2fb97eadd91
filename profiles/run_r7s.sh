# backward dH epilogue: operand and LN-backward sums released behind one fence
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stream.py tests/test_gpu_pairing.py -x -q > gpurun_out/r7s_pytest.txt 2>&1
echo "rc=$?" >> gpurun_out/r7s_pytest.txt
for v in pair nopair pair; do
  if [ $v = pair ]; then O=""; else O="--opt pair_recompute=0"; fi
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline $O > gpurun_out/r7s_bench_$v.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/r7s_bench_$v.json')); t=d['pipeline']['tasks']
print('$v', round(d['ms_per_step'],2), {k: round(v['median_us'],1) for k, v in t.items()}, 'frac', round(d['roofline']['frac'],4))" >> gpurun_out/r7s_summary.txt
done
timeout 300 python profiles/st_phases.py blocks=32 bwd=1 > gpurun_out/r7s_phases_bwd32.txt 2>&1
