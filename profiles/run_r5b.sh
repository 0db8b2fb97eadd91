#!/bin/bash
# stream-kernel phase timeline at HEAD (per-phase %globaltimer stamps), fwd and bwd
mkdir -p gpurun_out
timeout 300 python profiles/st_phases.py blocks=8 > gpurun_out/r5b_phases_fwd.txt 2>&1
timeout 300 python profiles/st_phases.py blocks=8 bwd=1 > gpurun_out/r5b_phases_bwd.txt 2>&1
timeout 300 python profiles/st_time.py 0 32 128 > gpurun_out/r5b_st_time.txt 2>&1
tail -4 gpurun_out/r5b_phases_fwd.txt gpurun_out/r5b_phases_bwd.txt gpurun_out/r5b_st_time.txt
