mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r7a_pytest_gpu.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/r7a_pytest_gpu.txt
timeout 300 python bench.py > gpurun_out/r7a_bench.json 2> gpurun_out/r7a_bench.err
echo "bench rc=$?"
