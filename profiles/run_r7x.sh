# HEAD validation after the gemm_tc bulk push and gemm_dw 128 x 256 tiles: full GPU suite, smoke, bench, C3 m = 4 / 8
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r7x_pytest_gpu.txt 2>&1
echo "rc=$?" >> gpurun_out/r7x_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r7x_smoke.txt 2>&1
timeout 300 python bench.py > gpurun_out/r7x_bench.json 2> gpurun_out/r7x_bench.err
for m in 4 8; do timeout 300 python bench.py --chunks $m --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r7x_c3_$m.json 2>/dev/null; done
timeout 900 python profiles/bench_c5.py --layers 48 --steps 2 --warmup 1 > gpurun_out/r7x_c5.json 2> gpurun_out/r7x_c5.err
tail -n 2 gpurun_out/r7x_pytest_gpu.txt; tail -1 gpurun_out/r7x_smoke.txt; cut -c1-200 gpurun_out/r7x_bench.json
