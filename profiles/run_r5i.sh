#!/bin/bash
mkdir -p gpurun_out
(echo "== vpx"; TGP_LIB=variants/libtgp_vpx.so timeout 120 python profiles/diag/determinism.py 4096 2 64 4 f 1 2>&1 | tail -2) > gpurun_out/r5i_det.txt 2>&1
cat gpurun_out/r5i_det.txt
