#!/bin/bash
# sanitizers on the small end-to-end cases, ncu launch list of the C2 bench step, ncu --set full of the
# stream kernel (F task) and the fused W_j + SGD kernel, SASS mnemonics of the product kernels
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck racecheck; do
  timeout 900 $CS --tool $tool --print-limit 20 --log-file gpurun_out/r5o_san_$tool.log python profiles/diag/sanitize_case.py > gpurun_out/r5o_san_${tool}_stdout.log 2>&1
  echo "rc=$?" >> gpurun_out/r5o_san_${tool}_stdout.log
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
    --log-file gpurun_out/r5o_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:task_stream_kernel -s 40 -c 1 \
    -o gpurun_out/r5o_stream python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r5o_ncu_stream.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:wgrad_sgd_kernel -s 2 -c 1 \
    -o gpurun_out/r5o_wgrad python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r5o_ncu_wgrad.log 2>&1
for t in memcheck synccheck racecheck; do echo "== $t"; tail -4 gpurun_out/r5o_san_$t.log; tail -6 gpurun_out/r5o_san_${t}_stdout.log; done
ls -la gpurun_out/ | tail -12
