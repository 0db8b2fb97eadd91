"""Per-kernel share of one step from an ncu launch list (gpu__time_duration.sum, --csv).
    python profiles/launch_share.py launches.csv [n_steps_in_file=2]   -> the last step's kernels"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
nsteps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
hdr, data = None, []
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d["Metric Name"] == "gpu__time_duration.sum":
            data.append(d)
last = data[len(data) - len(data) // nsteps:]
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
agg = collections.defaultdict(lambda: [0, 0.0])
for d in last:
    name = d["Kernel Name"].split("(")[0][:70]
    agg[name][0] += 1
    agg[name][1] += float(d["Metric Value"]) * scale.get(d["Metric Unit"], 1.0)
tot = sum(v[1] for v in agg.values())
print(f"kernels: {len(last)}   serialised device time: {tot / 1e3:.2f} ms")
for n, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{v / 1e3:9.3f} ms {100 * v / tot:5.1f}% {c:5d}  {n}")
