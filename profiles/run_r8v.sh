# throttle the hoisted F' of a pair (lane 2) so the critical B lane gets more HBM: pair_inflight sweep
mkdir -p gpurun_out
for v in 0 3 5 7 0 5; do
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --opt pair_inflight=$v > gpurun_out/r8v_tmp.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/r8v_tmp.json')); t=d['pipeline']['tasks']
print('pair_inflight=$v', round(d['ms_per_step'],2), {k: round(v['median_us'],1) for k, v in t.items()})" >> gpurun_out/r8v_summary.txt
done
cat gpurun_out/r8v_summary.txt
