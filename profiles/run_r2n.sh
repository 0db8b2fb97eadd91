OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q --timeout 300 > $OUT/pytest_gpu_r2n.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu_r2n.log
tail -2 $OUT/pytest_gpu_r2n.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > $OUT/bench_r2n.json 2> $OUT/bench_r2n.err; cat $OUT/bench_r2n.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 700 -c 400 --csv --log-file $OUT/launches_r2n.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $OUT/ncu_launch_r2n.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:task_stream_kernel -s 70 -c 1 -o $OUT/prof_stream_r2n python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $OUT/ncu_full_r2n.log 2>&1
tail -1 $OUT/ncu_full_r2n.log
