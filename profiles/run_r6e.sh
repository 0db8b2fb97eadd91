#!/bin/bash
(export TGP_LIB=$PWD/variants/timing/libtgp.so
CHUNKS=8 timeout 300 python profiles/gemm_timeline.py 4 2>&1 | head -9
CHUNKS=4 timeout 300 python profiles/gemm_timeline.py 4 2>&1 | head -9)
for m in 4 8 1; do
timeout 300 python bench.py --chunks $m --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r6e_m$m.json 2> gpurun_out/r6e_m$m.err
python - $m <<'PY'
import json,sys
d=json.loads(open(f"gpurun_out/r6e_m{sys.argv[1]}.json").read().strip().splitlines()[-1])
t=d["pipeline"]["tasks"]
print("m", sys.argv[1], round(d["ms_per_step"],2), "ms", {k: round(v["median_us"]) for k,v in t.items()}, d["roofline"]["frac"])
PY
done
timeout 900 python -m pytest -x -q tests/test_gpu_gemm.py tests/test_gpu_parity.py > gpurun_out/r6e_tests.txt 2>&1; tail -3 gpurun_out/r6e_tests.txt
