OUT=gpurun_out; mkdir -p $OUT
timeout 600 python bench.py > $OUT/bench_r2g.json 2> $OUT/bench_r2g.err; cat $OUT/bench_r2g.json; tail -2 $OUT/bench_r2g.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 0 > $OUT/bench_ref_r2g.json 2>&1; tail -1 $OUT/bench_ref_r2g.json
