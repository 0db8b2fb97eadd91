# gemm_tc skinny tiles (BN <= 64): 7 pipeline stages at BN = 64 (variant skinny7, 168 KB) vs 6 (HEAD, 160 KB); C3 m = 8 / 4
mkdir -p gpurun_out
for v in default skinny7 default skinny7; do
  if [ $v = default ]; then L=""; else L="variants/$v/libtgp.so"; fi
  for m in 8; do
    TGP_LIB=$L timeout 300 python bench.py --chunks $m --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r8b_bench_${v}_$m.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/r8b_bench_${v}_$m.json')); t=d['pipeline']['tasks']
print('$v m=$m', round(d['ms_per_step'],2), {k: round(v['median_us'],1) for k, v in t.items()})" >> gpurun_out/r8b_summary.txt
  done
done
cat gpurun_out/r8b_summary.txt
