# final C3 sweep at HEAD + C4 U-MLP bench
mkdir -p gpurun_out
for m in 32 8 4 1; do for ck in except_last always never; do
  timeout 300 python bench.py --chunks $m --checkpoint $ck --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r8w_c3_${m}_$ck.json 2>/dev/null
done; done
timeout 600 python profiles/bench_c4.py > gpurun_out/r8w_c4.json 2> gpurun_out/r8w_c4.err
tail -c 400 gpurun_out/r8w_c4.json
