#!/bin/bash
# multi-rank code paths at HEAD on one GPU (8 and 2 processes; a code-path check, not a measurement)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_multiproc.py -x -q --timeout 1000 -k c2_n8 > gpurun_out/r8u_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r8u_pytest.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29621 \
   bench.py --gpus 8 --steps 3 --warmup 3 > gpurun_out/r8u_bench_n8_1gpu.json 2> gpurun_out/r8u_bench_n8.err
echo "bench rc=$?" >> gpurun_out/r8u_bench_n8.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29622 \
   bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/r8u_bench_n2_1gpu.json 2> gpurun_out/r8u_bench_n2.err
tail -5 gpurun_out/r8u_pytest.log; cut -c1-600 gpurun_out/r8u_bench_n8_1gpu.json gpurun_out/r8u_bench_n2_1gpu.json; tail -3 gpurun_out/r8u_bench_n8.err
