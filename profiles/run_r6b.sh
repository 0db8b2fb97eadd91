#!/bin/bash
# C3 points under gemm_tc stage-budget variants
mkdir -p gpurun_out
for lib in default w128_6 sk_6; do
  for m in 1 4 8; do
    if [ $lib = default ]; then unset TGP_LIB; else export TGP_LIB=$PWD/variants/$lib/libtgp.so; fi
    timeout 300 python bench.py --chunks $m --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r6b_${lib}_m$m.json 2> gpurun_out/r6b_${lib}_m$m.err
    python - $lib $m <<'PY'
import json,sys
d=json.loads(open(f"gpurun_out/r6b_{sys.argv[1]}_m{sys.argv[2]}.json").read().strip().splitlines()[-1])
t=d["pipeline"]["tasks"]
print(sys.argv[1], "m", sys.argv[2], round(d["ms_per_step"],2), "ms", {k: round(v["median_us"]) for k,v in t.items()}, d["roofline"]["frac"], d["roofline"].get("kernel",""))
PY
  done
done
