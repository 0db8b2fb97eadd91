# gemm_tc split-K partials: bulk DSMEM copies (variant bulkpush) vs per-float4 st.async (HEAD), C3 m = 4 / 8
mkdir -p gpurun_out
TGP_LIB=variants/bulkpush/libtgp.so timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_parity.py -x -q > gpurun_out/r7t_pytest_bulk.txt 2>&1
echo "rc=$?" >> gpurun_out/r7t_pytest_bulk.txt
for v in default bulkpush default bulkpush; do
  if [ $v = default ]; then L=""; else L="variants/$v/libtgp.so"; fi
  for m in 4 8; do
    TGP_LIB=$L timeout 300 python bench.py --chunks $m --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r7t_bench_${v}_$m.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/r7t_bench_${v}_$m.json')); t=d['pipeline']['tasks']
print('$v m=$m', round(d['ms_per_step'],2), {k: round(v['median_us'],1) for k, v in t.items()})" >> gpurun_out/r7t_summary.txt
  done
done
cat gpurun_out/r7t_summary.txt; tail -n 2 gpurun_out/r7t_pytest_bulk.txt
