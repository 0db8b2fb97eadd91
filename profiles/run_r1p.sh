OUT=gpurun_out; mkdir -p $OUT
timeout 300 python -m pytest tests/test_gpu_stream.py -x -q --timeout 120 > $OUT/pytest_stream_r1p.log 2>&1; echo "rc=$?" >> $OUT/pytest_stream_r1p.log
tail -3 $OUT/pytest_stream_r1p.log
timeout 600 python bench.py > $OUT/bench_r1p.json 2> $OUT/bench_r1p.err; cat $OUT/bench_r1p.json; tail -3 $OUT/bench_r1p.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 1200 -c 500 --csv --log-file $OUT/launches_r1p.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $OUT/ncu_launch_r1p.log 2>&1
tail -2 $OUT/ncu_launch_r1p.log
