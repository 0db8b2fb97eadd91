#!/bin/bash
# f1 ablation toggles: parity tests, then the Table 1 measurement (paper's setting and C4's)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ablation.py tests/test_gpu_parity.py -q -x -k "ablation or c4 or c1" 2>&1 | tail -5
timeout 600 python profiles/ablation_f1.py --d 2048 --batch 128 --chunks 8 --parts 4 --steps 10 2>&1 | tee gpurun_out/r3g_ablation_paper.txt
timeout 600 python profiles/ablation_f1.py --d 2048 --batch 256 --chunks 32 --parts 8 --steps 5 2>&1 | tee gpurun_out/r3g_ablation_c4.txt
