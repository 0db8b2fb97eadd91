#!/bin/bash
timeout 900 python -m pytest -x -q tests/test_gpu_gemm.py tests/test_gpu_parity.py tests/test_gpu_gpt2.py > gpurun_out/r6j_tests.txt 2>&1; tail -2 gpurun_out/r6j_tests.txt
for m in 1 4 8; do
timeout 300 python bench.py --chunks $m --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r6j_m$m.json 2> gpurun_out/r6j_m$m.err
python - $m <<'PY'
import json,sys
d=json.loads(open(f"gpurun_out/r6j_m{sys.argv[1]}.json").read().strip().splitlines()[-1])
t=d["pipeline"]["tasks"]
print("m", sys.argv[1], round(d["ms_per_step"],2), "ms", {k: round(v["median_us"]) for k,v in t.items()}, d["roofline"]["frac"])
PY
done
timeout 900 python profiles/bench_c5.py --layers 48 --steps 2 --warmup 1 > gpurun_out/r6j_c5.json 2> gpurun_out/r6j_c5.err; tail -1 gpurun_out/r6j_c5.json | cut -c1-400
