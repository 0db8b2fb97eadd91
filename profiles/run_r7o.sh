# HEAD record: full GPU suite, smoke, bench (default args), reference arm, phase stamps
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r7o_pytest_gpu.txt 2>&1
echo "rc=$?" >> gpurun_out/r7o_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r7o_smoke.txt 2>&1
timeout 300 python bench.py > gpurun_out/r7o_bench.json 2> gpurun_out/r7o_bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r7o_bench_reference.json 2> gpurun_out/r7o_bench_reference.err
timeout 300 python profiles/st_phases.py blocks=8 > gpurun_out/r7o_phases_fwd.txt 2>&1
tail -n 2 gpurun_out/r7o_pytest_gpu.txt; cat gpurun_out/r7o_smoke.txt | tail -1; cut -c1-300 gpurun_out/r7o_bench.json; cut -c1-300 gpurun_out/r7o_bench_reference.json
