mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_async.py -x -q > gpurun_out/r7b_pytest_async.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/r7b_pytest_async.txt
for ch in 4 8; do for sk in 4 8; do
  echo "=== CHUNKS=$ch splitk=$sk" >> gpurun_out/r7b_gemm_timeline.txt
  CHUNKS=$ch TGP_LIB=variants/timing/libtgp.so timeout 300 python profiles/gemm_timeline.py $sk >> gpurun_out/r7b_gemm_timeline.txt 2>&1
done; done
