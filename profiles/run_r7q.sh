# backward copies: tcgen05.st.16x256b.x4 (2 per tile per warp instead of 8 x1)
mkdir -p gpurun_out
(cd profiles && timeout 60 ./ldsm_probe) > gpurun_out/r7q_ldsm_probe.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_stream.py tests/test_gpu_pairing.py -x -q > gpurun_out/r7q_pytest.txt 2>&1
echo "rc=$?" >> gpurun_out/r7q_pytest.txt
for v in pair nopair pair; do
  if [ $v = pair ]; then O=""; else O="--opt pair_recompute=0"; fi
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline $O > gpurun_out/r7q_bench_$v.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/r7q_bench_$v.json')); t=d['pipeline']['tasks']
print('$v', round(d['ms_per_step'],2), {k: round(v['median_us'],1) for k, v in t.items()}, 'frac', round(d['roofline']['frac'],4))" >> gpurun_out/r7q_summary.txt
done
timeout 300 python profiles/st_phases.py blocks=32 bwd=1 > gpurun_out/r7q_phases_bwd32.txt 2>&1
head -2 gpurun_out/r7q_ldsm_probe.txt; cat gpurun_out/r7q_summary.txt; tail -n 2 gpurun_out/r7q_pytest.txt; tail -n 1 gpurun_out/r7q_phases_bwd32.txt
