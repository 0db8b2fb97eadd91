#!/bin/bash
# One gpurun session: tests, smoke, bench, ncu launch list, ncu full capture of the dominant GEMM.
# Usage (from the repo root on the GPU box): bash profiles/run_gpu_round.sh <tag>
TAG=${1:-r1}
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q --timeout 300 > $OUT/pytest_gpu_$TAG.log 2>&1
echo "pytest rc=$?" >> $OUT/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1
timeout 900 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 34500 -c 3000 --csv \
    --log-file $OUT/launches_$TAG.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $OUT/ncu_launch_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 200 -c 2 \
    -o $OUT/prof_gemm_$TAG python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $OUT/ncu_full_$TAG.log 2>&1
tail -3 $OUT/pytest_gpu_$TAG.log; cat $OUT/smoke_$TAG.log | tail -2; cat $OUT/bench_$TAG.json; tail -3 $OUT/bench_$TAG.err
