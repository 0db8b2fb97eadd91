"""Stage-boundary transport sweep: per-message device time
of the SM push kernel (mode 0) and the copy engine (mode 1), 4 KiB .. 64 MiB, for every ordered
device pair on the box (a one-GPU box measures the local path only).
    python profiles/transport_sweep.py [reps=50]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2004_09910_b200 import bench_transport  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 50
ndev = torch.cuda.device_count()
pairs = [(a, b) for a in range(ndev) for b in range(ndev)] if ndev > 1 else [(0, 0)]
rows = []
print(f"{'src':>3} {'dst':>3} {'bytes':>10} | {'push us':>8} {'push GB/s':>9} {'pingpong':>8} | {'CE us':>8} {'CE GB/s':>8} {'pingpong':>8} | pick")
for a, b in pairs:
    for k in range(12, 27, 2):
        n = 1 << k
        r = {"src": a, "dst": b, "bytes": n}
        for mode, name in ((0, "push"), (1, "ce")):
            us, pp = bench_transport(a, b, n, mode, reps=reps)
            r[name + "_us"], r[name + "_pingpong_us"], r[name + "_gbs"] = us, pp, n / us / 1e3
        r["pick"] = "push" if r["push_us"] <= r["ce_us"] else "ce"
        rows.append(r)
        print(f"{a:>3} {b:>3} {n:>10} | {r['push_us']:8.2f} {r['push_gbs']:9.1f} {r['push_pingpong_us']:8.2f} | "
              f"{r['ce_us']:8.2f} {r['ce_gbs']:8.1f} {r['ce_pingpong_us']:8.2f} | {r['pick']}", flush=True)
print(json.dumps({"transport_sweep": rows}))
