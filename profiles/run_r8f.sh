# HEAD full GPU suite (memory-plan test updated for per-layer pairing; new per-layer pairing tests) + smoke
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r8f_pytest_gpu.txt 2>&1
echo "rc=$?" >> gpurun_out/r8f_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r8f_smoke.txt 2>&1
tail -n 3 gpurun_out/r8f_pytest_gpu.txt; tail -n 1 gpurun_out/r8f_smoke.txt
