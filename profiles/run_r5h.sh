#!/bin/bash
mkdir -p gpurun_out
for cfg in "4096 4 512 32" "1024 4 128 8" "4096 2 64 4"; do timeout 120 python profiles/diag/determinism.py $cfg; done > gpurun_out/r5h_det.txt 2>&1
cat gpurun_out/r5h_det.txt
