#!/bin/bash
# C3 sweep at HEAD (BASELINE configs[2] at n = 1): checkpoint mode x m, C2 model, B = 512
mkdir -p gpurun_out
for m in 32 8 4 1; do for ck in except_last always never; do
  timeout 300 python bench.py --chunks $m --checkpoint $ck --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r6o_c3_${m}_${ck}.json 2>/dev/null
  python -c "
import json
d=json.load(open('gpurun_out/r6o_c3_${m}_${ck}.json'))
t=d['pipeline']['tasks']
print(f\"m={d['config']['chunks']:3d} {d['config']['checkpoint']:12s} {d['ms_per_step']:8.2f} ms/step {d['value']:8.0f} samples/s  F {t.get('F',{}).get('median_us',0):7.0f} us  F' {t.get(\\\"F'\\\",{}).get('median_us',0):7.0f} us  B {t.get('B',{}).get('median_us',0):7.0f} us  W {t.get('W',{}).get('median_us',0):7.0f} us  stream-F frac {d['roofline']['frac']:.3f} ({d['roofline']['kernel'][:22]})\")
" >> gpurun_out/r6o_c3_sweep.txt 2>&1
done; done
cat gpurun_out/r6o_c3_sweep.txt
timeout 900 python profiles/bench_c5.py --layers 48 --steps 2 --warmup 1 > gpurun_out/r6o_c5.json 2> gpurun_out/r6o_c5.err; tail -1 gpurun_out/r6o_c5.json | cut -c1-500
