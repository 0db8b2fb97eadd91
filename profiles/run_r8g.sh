# end-of-round record at HEAD: bench (default), reference arm, C3 sweep (m x checkpoint), ncu launch list of one C2 step
mkdir -p gpurun_out
timeout 300 python bench.py > gpurun_out/r8g_bench.json 2> gpurun_out/r8g_bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r8g_bench_reference.json 2> gpurun_out/r8g_bench_reference.err
for m in 32 8 4 1; do for ck in except_last always never; do
  timeout 300 python bench.py --chunks $m --checkpoint $ck --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r8g_c3_${m}_$ck.json 2>/dev/null
done; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
    --log-file gpurun_out/r8g_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
cut -c1-200 gpurun_out/r8g_bench.json
