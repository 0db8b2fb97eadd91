# HEAD: per-layer F'/B pairing + bulk push, dW tiles back to 128 x 128: full GPU suite twice, C5 full, C3 m = 4 / 8
mkdir -p gpurun_out
for i in 1 2; do
  timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r8e_pytest_gpu_$i.txt 2>&1
  echo "rc=$?" >> gpurun_out/r8e_pytest_gpu_$i.txt
  tail -n 2 gpurun_out/r8e_pytest_gpu_$i.txt
done
timeout 900 python profiles/bench_c5.py --layers 48 --steps 2 --warmup 1 > gpurun_out/r8e_c5.json 2> gpurun_out/r8e_c5.err
tail -c 300 gpurun_out/r8e_c5.json; tail -2 gpurun_out/r8e_c5.err
for m in 4 8; do for ck in except_last always never; do
  timeout 300 python bench.py --chunks $m --checkpoint $ck --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r8e_c3_${m}_$ck.json 2>/dev/null
done; done
timeout 300 python bench.py > gpurun_out/r8e_bench.json 2>/dev/null; cut -c1-150 gpurun_out/r8e_bench.json
