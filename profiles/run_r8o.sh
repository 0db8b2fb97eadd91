# is the backward straggler always the same CTA?  three lag runs
mkdir -p gpurun_out
for i in 1 2 3; do
  timeout 300 python profiles/st_phases.py blocks=32 bwd=1 lag=1 > gpurun_out/r8o_bwd_lag_$i.txt 2>&1
  grep -A 4 "CTA (cluster" gpurun_out/r8o_bwd_lag_$i.txt; grep "lag by" gpurun_out/r8o_bwd_lag_$i.txt
done
