# HEAD: copy-warp throttle on the full grid; full GPU suite; NVTX range capture evidence
mkdir -p gpurun_out
timeout 300 python bench.py > gpurun_out/r7g_bench.json 2> gpurun_out/r7g_bench.err
timeout 300 ncu --nvtx --nvtx-include "W j=1/" --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/r7g_nvtx_W.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline > /dev/null 2>&1
timeout 300 ncu --nvtx --nvtx-include "F i=5 j=1/" --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/r7g_nvtx_F5.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline > /dev/null 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r7g_pytest_gpu.txt 2>&1
echo "rc=$?" >> gpurun_out/r7g_pytest_gpu.txt
cut -c1-600 gpurun_out/r7g_bench.json; tail -n 2 gpurun_out/r7g_pytest_gpu.txt
