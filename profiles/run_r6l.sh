#!/bin/bash
for m in 4 8; do
timeout 300 python bench.py --chunks $m --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r6l_m$m.json 2> gpurun_out/r6l_m$m.err
python - $m <<'PY'
import json,sys
d=json.loads(open(f"gpurun_out/r6l_m{sys.argv[1]}.json").read().strip().splitlines()[-1])
t=d["pipeline"]["tasks"]
print("m", sys.argv[1], round(d["ms_per_step"],2), "ms", {k: round(v["median_us"]) for k,v in t.items()}, d["roofline"]["frac"])
PY
done
timeout 900 python -m pytest -x -q tests/test_gpu_parity.py tests/test_gpu_stream.py tests/test_gpu_ln_dropout.py > gpurun_out/r6l_tests.txt 2>&1; tail -2 gpurun_out/r6l_tests.txt
