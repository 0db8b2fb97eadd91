# stream kernel acquire-side experiment: ld.acquire re-read (default) vs fence.acq_rel (old) vs per-warp release
mkdir -p gpurun_out
for v in default fenceacq warprel default fenceacq warprel; do
  if [ $v = default ]; then L=""; else L="variants/$v/libtgp.so"; fi
  TGP_LIB=$L timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r7c_bench_$v.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/r7c_bench_$v.json')); t=d['pipeline']['tasks']
print('$v', round(d['ms_per_step'],2), 'F', t['F']['median_us'], 'Fp', t[\"F'\"]['median_us'], 'B', t['B']['median_us'], 'frac', round(d['roofline']['frac'],4))" >> gpurun_out/r7c_summary.txt
done
for v in default warprel; do
  if [ $v = default ]; then L=""; else L="variants/$v/libtgp.so"; fi
  TGP_LIB=$L timeout 600 python -m pytest tests/test_gpu_stream.py tests/test_gpu_pairing.py -x -q > gpurun_out/r7c_pytest_$v.txt 2>&1
  echo "rc=$?" >> gpurun_out/r7c_pytest_$v.txt
done
cat gpurun_out/r7c_summary.txt
