#!/bin/bash
timeout 2400 python -m pytest -q -m gpu tests/ -x > gpurun_out/r6i_pytest_gpu.txt 2>&1; tail -3 gpurun_out/r6i_pytest_gpu.txt
timeout 300 python bench.py > gpurun_out/r6i_bench.json 2> gpurun_out/r6i_bench.err; tail -1 gpurun_out/r6i_bench.json | cut -c1-300
