# final HEAD record: bench (default), smoke, C5 full
mkdir -p gpurun_out
timeout 300 python bench.py > gpurun_out/r8k_bench.json 2> gpurun_out/r8k_bench.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r8k_smoke.txt 2>&1
timeout 900 python profiles/bench_c5.py --layers 48 --steps 2 --warmup 1 > gpurun_out/r8k_c5.json 2> gpurun_out/r8k_c5.err
cut -c1-200 gpurun_out/r8k_bench.json; tail -1 gpurun_out/r8k_smoke.txt; tail -c 250 gpurun_out/r8k_c5.json
