# gemm_dw tile width: 128 x 256 (variant dwbn256) vs 128 x 128 (HEAD) on the C5 8-layer step and C2
mkdir -p gpurun_out
for v in default dwbn256 default dwbn256; do
  if [ $v = default ]; then L=""; else L="variants/$v/libtgp.so"; fi
  TGP_LIB=$L timeout 600 python profiles/bench_c5.py --layers 8 --seqs 8 --chunks 8 --steps 3 --warmup 2 > gpurun_out/r7w_c5_$v.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/r7w_c5_$v.json').read().strip().splitlines()[-1]); print('$v C5-8L', round(d['ms_per_step'],2), 'ms', round(d['model_tflops'],1), 'TF/s')" >> gpurun_out/r7w_summary.txt
done
TGP_LIB=variants/dwbn256/libtgp.so timeout 600 python -m pytest tests/test_gpu_gemm.py -x -q -k "dw" > gpurun_out/r7w_pytest.txt 2>&1
echo "rc=$?" >> gpurun_out/r7w_pytest.txt
cat gpurun_out/r7w_summary.txt; tail -n 2 gpurun_out/r7w_pytest.txt
