# final HEAD validation: full GPU suite, smoke, bench, reference arm
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r8s_pytest_gpu.txt 2>&1
echo "rc=$?" >> gpurun_out/r8s_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r8s_smoke.txt 2>&1
timeout 300 python bench.py > gpurun_out/r8s_bench.json 2> gpurun_out/r8s_bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r8s_bench_reference.json 2> gpurun_out/r8s_bench_reference.err
tail -n 2 gpurun_out/r8s_pytest_gpu.txt; tail -n 1 gpurun_out/r8s_smoke.txt; cut -c1-160 gpurun_out/r8s_bench.json
