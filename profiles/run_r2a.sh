OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q --timeout 300 > $OUT/pytest_gpu_r2a.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu_r2a.log
tail -3 $OUT/pytest_gpu_r2a.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > $OUT/bench_r2a.json 2> $OUT/bench_r2a.err; cat $OUT/bench_r2a.json; tail -2 $OUT/bench_r2a.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 1200 -c 500 --csv --log-file $OUT/launches_r2a.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $OUT/ncu_launch_r2a.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:task_stream_kernel -s 70 -c 1 -o $OUT/prof_stream_r2a python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $OUT/ncu_full_r2a.log 2>&1
tail -2 $OUT/ncu_launch_r2a.log $OUT/ncu_full_r2a.log
