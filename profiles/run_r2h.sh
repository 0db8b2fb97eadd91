OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 2>&1 | tail -2
for m in 32 8 4 1; do for ck in except_last never always; do
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --chunks $m --checkpoint $ck 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(f\"m={d['config']['chunks']:3d} {d['config']['checkpoint']:12s} {d['value']:9.1f} samples/s  {d['ms_per_step']:8.2f} ms/step  kernel={d['roofline']['kernel'][:40]} frac={d['roofline']['frac']:.3f}\")" >> $OUT/c3_sweep_r2h.txt
done; done
cat $OUT/c3_sweep_r2h.txt
