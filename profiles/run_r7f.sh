# copy-warp throttle during a phase's MMA window (variant) vs HEAD; nvtx evidence via ncu range filter
mkdir -p gpurun_out
for v in default throttle default throttle; do
  if [ $v = default ]; then L=""; else L="variants/$v/libtgp.so"; fi
  TGP_LIB=$L timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r7f_bench_$v.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/r7f_bench_$v.json')); t=d['pipeline']['tasks']
print('$v', round(d['ms_per_step'],2), 'F', t['F']['median_us'], 'Fp', t[\"F'\"]['median_us'], 'B', t['B']['median_us'], 'frac', round(d['roofline']['frac'],4))" >> gpurun_out/r7f_summary.txt
done
TGP_LIB=variants/throttle/libtgp.so timeout 600 python -m pytest tests/test_gpu_stream.py tests/test_gpu_pairing.py -x -q > gpurun_out/r7f_pytest_throttle.txt 2>&1
echo "rc=$?" >> gpurun_out/r7f_pytest_throttle.txt
timeout 300 ncu --nvtx --nvtx-include "regex:^W j=1" --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/r7f_nvtx_W.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline > /dev/null 2>&1
timeout 300 ncu --nvtx --nvtx-include "regex:^F i=5 j=1" --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/r7f_nvtx_F5.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline > /dev/null 2>&1
cat gpurun_out/r7f_summary.txt; tail -n 2 gpurun_out/r7f_pytest_throttle.txt
