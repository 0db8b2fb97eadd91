# backward: dH column sums deferred past the next dG epilogue's signal -- tests + bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stream.py tests/test_gpu_pairing.py tests/test_gpu_fused_send.py tests/test_gpu_fused_sgd.py tests/test_gpu_parity.py -x -q > gpurun_out/r8m_pytest.txt 2>&1
echo "rc=$?" >> gpurun_out/r8m_pytest.txt
tail -n 2 gpurun_out/r8m_pytest.txt
for v in pair nopair pair nopair; do
  if [ $v = pair ]; then O=""; else O="--opt pair_recompute=0"; fi
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline $O > gpurun_out/r8m_bench_$v.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/r8m_bench_$v.json')); t=d['pipeline']['tasks']
print('$v', round(d['ms_per_step'],2), {k: round(v['median_us'],1) for k, v in t.items()}, d['clocks']['reasons'])" >> gpurun_out/r8m_summary.txt
done
cat gpurun_out/r8m_summary.txt
