OUT=gpurun_out; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/gpu_r1i.txt
timeout 900 python -m pytest tests -m gpu -q --timeout 300 > $OUT/pytest_gpu_r1i.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu_r1i.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_r1i.log 2>&1
timeout 600 python bench.py > $OUT/bench_r1i.json 2> $OUT/bench_r1i.err
timeout 600 python bench.py --no-cpu-baseline --opt persistent=1 > $OUT/bench_r1i_pt.json 2> $OUT/bench_r1i_pt.err
timeout 600 python bench.py --no-cpu-baseline --checkpoint never > $OUT/bench_r1i_never.json 2>> $OUT/bench_r1i.err
for sk in 0 4 8; do timeout 120 python profiles/gemm_chain.py $sk >> $OUT/chain_r1i.txt 2>&1; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 34500 -c 3000 --csv --log-file $OUT/launches_r1i.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $OUT/ncu_launch_r1i.log 2>&1
tail -3 $OUT/pytest_gpu_r1i.log; tail -2 $OUT/smoke_r1i.log; cat $OUT/bench_r1i*.json $OUT/chain_r1i.txt
