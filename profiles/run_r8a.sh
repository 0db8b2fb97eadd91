# stress: the test that hit a one-off illegal address in r7x, 25 times at HEAD, then the C5 / GEMM tests 3 times
mkdir -p gpurun_out
pass=0; fail=0
for i in $(seq 1 25); do
  if timeout 120 python -m pytest tests/test_gpu_gpt2.py -q -k "wider_multi_tile" > gpurun_out/r8a_run.txt 2>&1; then pass=$((pass+1)); else fail=$((fail+1)); cp gpurun_out/r8a_run.txt gpurun_out/r8a_fail_$i.txt; fi
done
echo "wider_multi_tile: pass $pass fail $fail" > gpurun_out/r8a_summary.txt
for i in 1 2 3; do
  timeout 600 python -m pytest tests/test_gpu_gpt2.py tests/test_gpu_gemm.py tests/test_gpu_parity.py -q > gpurun_out/r8a_suite_$i.txt 2>&1
  echo "suite $i rc=$? $(tail -n 1 gpurun_out/r8a_suite_$i.txt)" >> gpurun_out/r8a_summary.txt
done
cat gpurun_out/r8a_summary.txt
