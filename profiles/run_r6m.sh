#!/bin/bash
for lib in default lnb16; do
if [ $lib = default ]; then unset TGP_LIB; else export TGP_LIB=$PWD/variants/$lib/libtgp.so; fi
for m in 4 8; do
timeout 300 python bench.py --chunks $m --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r6m_${lib}_m$m.json 2> gpurun_out/r6m_m$m.err
python - $m $lib <<'PY'
import json,sys
d=json.loads(open(f"gpurun_out/r6m_{sys.argv[2]}_m{sys.argv[1]}.json").read().strip().splitlines()[-1])
t=d["pipeline"]["tasks"]
print(sys.argv[2], "m", sys.argv[1], round(d["ms_per_step"],2), "ms", {k: round(v["median_us"]) for k,v in t.items()}, d["roofline"]["frac"])
PY
done; done
export TGP_LIB=$PWD/variants/lnb16/libtgp.so
timeout 900 python -m pytest -x -q tests/test_gpu_parity.py > gpurun_out/r6m_tests.txt 2>&1; tail -1 gpurun_out/r6m_tests.txt
