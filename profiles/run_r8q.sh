# HEAD: copy throttle only in the forward; full GPU suite, bench, never-mode bench, C3 sweep m = 32
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r8q_pytest_gpu.txt 2>&1
echo "rc=$?" >> gpurun_out/r8q_pytest_gpu.txt
tail -n 2 gpurun_out/r8q_pytest_gpu.txt
timeout 300 python bench.py > gpurun_out/r8q_bench.json 2> gpurun_out/r8q_bench.err
for ck in always never; do timeout 300 python bench.py --checkpoint $ck --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r8q_bench_$ck.json 2>/dev/null; done
python -c "
import json
for f in ('r8q_bench','r8q_bench_always','r8q_bench_never'):
    d=json.load(open('gpurun_out/'+f+'.json')); t=d['pipeline']['tasks']
    print(f, round(d['value']), round(d['ms_per_step'],2), {k: round(v['median_us'],1) for k, v in t.items()}, round(d['roofline']['frac'],3), d['clocks']['reasons'])"
