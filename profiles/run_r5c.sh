#!/bin/bash
mkdir -p gpurun_out
timeout 300 python profiles/st_sweep.py stream_inflight=0,1,2,3,4,5,6,8 > gpurun_out/r5c_sweep.txt 2>&1
timeout 300 python profiles/st_phases.py blocks=8 inflight=3 > gpurun_out/r5c_phases_fwd_if3.txt 2>&1
cat gpurun_out/r5c_sweep.txt; tail -3 gpurun_out/r5c_phases_fwd_if3.txt
