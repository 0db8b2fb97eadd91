mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pairing.py -q > gpurun_out/r8l_pytest_pairing.txt 2>&1
echo "rc=$?" >> gpurun_out/r8l_pytest_pairing.txt
tail -n 2 gpurun_out/r8l_pytest_pairing.txt
