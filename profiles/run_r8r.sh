# per-CTA lag of the last PAIRED backward task (half grid beside F') and the unpaired one for comparison
mkdir -p gpurun_out
timeout 300 python profiles/st_phases.py blocks=32 bwd=1 paired=1 lag=1 > gpurun_out/r8r_bwd_paired_lag.txt 2>&1
timeout 300 python profiles/st_phases.py blocks=32 bwd=1 lag=1 > gpurun_out/r8r_bwd_lag.txt 2>&1
for f in gpurun_out/r8r_bwd_paired_lag.txt gpurun_out/r8r_bwd_lag.txt; do echo "== $f"; grep -A 5 "CTA (cluster" $f; grep "lag by rank\|total" $f; done
