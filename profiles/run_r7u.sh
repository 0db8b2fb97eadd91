# experiment: F task without its off-critical-path stores (a, LN-output stash, per-block y) -- does the operand
# release (MEMBAR) wait for them?  (variant results are garbage; timing only)
mkdir -p gpurun_out
for v in default nostash default nostash; do
  if [ $v = default ]; then L=""; else L="variants/$v/libtgp.so"; fi
  TGP_LIB=$L timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --opt pair_recompute=0 > gpurun_out/r7u_bench_$v.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/r7u_bench_$v.json')); t=d['pipeline']['tasks']
print('$v', round(d['ms_per_step'],2), {k: round(v['median_us'],1) for k, v in t.items()}, 'F kernel', round(d['roofline']['avg_launch_us'],1))" >> gpurun_out/r7u_summary.txt
done
cat gpurun_out/r7u_summary.txt
