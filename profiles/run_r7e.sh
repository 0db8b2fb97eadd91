# per-k-block activation barriers in the stream kernel
mkdir -p gpurun_out
for i in 1 2; do
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r7e_bench_$i.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/r7e_bench_$i.json')); t=d['pipeline']['tasks']
print('bfk', round(d['ms_per_step'],2), 'F', t['F']['median_us'], 'Fp', t[\"F'\"]['median_us'], 'B', t['B']['median_us'], 'frac', round(d['roofline']['frac'],4))" >> gpurun_out/r7e_summary.txt
done
timeout 600 python -m pytest tests/test_gpu_stream.py tests/test_gpu_pairing.py tests/test_gpu_fused_send.py -x -q > gpurun_out/r7e_pytest.txt 2>&1
echo "rc=$?" >> gpurun_out/r7e_pytest.txt
cat gpurun_out/r7e_summary.txt; tail -n 3 gpurun_out/r7e_pytest.txt
