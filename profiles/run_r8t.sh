# knob sweep at HEAD: stream_inflight and stream_poll_ns on the C2 bench
mkdir -p gpurun_out
for o in "" "--opt stream_inflight=6" "--opt stream_inflight=8" "--opt stream_poll_ns=16" "--opt stream_poll_ns=64" ""; do
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline $o > gpurun_out/r8t_tmp.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/r8t_tmp.json')); t=d['pipeline']['tasks']
print('[$o]', round(d['ms_per_step'],2), {k: round(v['median_us'],1) for k, v in t.items()})" >> gpurun_out/r8t_summary.txt
done
cat gpurun_out/r8t_summary.txt
