#!/bin/bash
for lib in default wg7 wg5 we8; do
if [ $lib = default ]; then unset TGP_LIB; else export TGP_LIB=$PWD/variants/$lib/libtgp.so; fi
timeout 300 python bench.py --chunks 1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r6n_${lib}_m1.json 2>/dev/null
timeout 600 python profiles/bench_c5.py --layers 8 --seqs 16 --chunks 16 --steps 3 --warmup 1 > gpurun_out/r6n_${lib}_c5.json 2>/dev/null
python - $lib <<'PY'
import json,sys
l=sys.argv[1]
d=json.loads(open(f"gpurun_out/r6n_{l}_m1.json").read().strip().splitlines()[-1])
c=json.loads(open(f"gpurun_out/r6n_{l}_c5.json").read().strip().splitlines()[-1])
print(l, "m1", round(d["ms_per_step"],2), {k: round(v["median_us"]) for k,v in d["pipeline"]["tasks"].items()}, "c5-8L", round(c["ms_per_step"],1), "ms", round(c["model_tflops"]), "TF/s")
PY
done
