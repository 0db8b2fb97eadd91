#!/bin/bash
export TGP_LIB=$PWD/variants/timing/libtgp.so
CHUNKS=8 timeout 300 python profiles/gemm_timeline.py 4 2>&1 | head -12
CHUNKS=4 timeout 300 python profiles/gemm_timeline.py 4 2>&1 | head -12
