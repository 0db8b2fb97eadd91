# copy-warp throttle off for the backward (variant nobwdthr) vs HEAD: unpaired / paired C2 and backward straggler lag
mkdir -p gpurun_out
for v in default nobwdthr default nobwdthr; do
  if [ $v = default ]; then L=""; else L="variants/$v/libtgp.so"; fi
  for o in pair nopair; do
    if [ $o = pair ]; then O=""; else O="--opt pair_recompute=0"; fi
    TGP_LIB=$L timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline $O > gpurun_out/r8p_bench_${v}_$o.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/r8p_bench_${v}_$o.json')); t=d['pipeline']['tasks']
print('$v $o', round(d['ms_per_step'],2), {k: round(v['median_us'],1) for k, v in t.items()})" >> gpurun_out/r8p_summary.txt
  done
done
TGP_LIB=variants/nobwdthr/libtgp.so timeout 300 python profiles/st_phases.py blocks=32 bwd=1 lag=1 > gpurun_out/r8p_bwd_lag_nothr.txt 2>&1
cat gpurun_out/r8p_summary.txt; grep -A 3 "CTA (cluster" gpurun_out/r8p_bwd_lag_nothr.txt; grep "lag by rank\|total" gpurun_out/r8p_bwd_lag_nothr.txt
