# which change breaks test_c5_wider_multi_tile: gemm_dw 128 x 256 tiles (HEAD) vs 128 x 128 (variant dw128)
mkdir -p gpurun_out
for v in default dw128; do
  if [ $v = default ]; then L=""; else L="variants/$v/libtgp.so"; fi
  TGP_LIB=$L timeout 600 python -m pytest tests/test_gpu_gpt2.py -x -q > gpurun_out/r7y_pytest_$v.txt 2>&1
  echo "$v rc=$?" >> gpurun_out/r7y_pytest_$v.txt
  tail -n 2 gpurun_out/r7y_pytest_$v.txt
done
