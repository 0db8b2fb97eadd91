# which CTAs set the backward phase time (per-CTA lag of MMA completion and of the last weight tile)
mkdir -p gpurun_out
timeout 300 python profiles/st_phases.py blocks=32 bwd=1 lag=1 > gpurun_out/r8n_bwd_lag.txt 2>&1
timeout 300 python profiles/st_phases.py blocks=32 lag=1 > gpurun_out/r8n_fwd_lag.txt 2>&1
tail -n 16 gpurun_out/r8n_bwd_lag.txt; tail -n 16 gpurun_out/r8n_fwd_lag.txt
