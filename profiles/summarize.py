"""Summarise ncu outputs (run here, on the CPU box) into profiles/<tag>_*.txt.

    python profiles/summarize.py <tag> [launches.csv] [prof.ncu-rep]

launch list  -> per-kernel count / total / average device time and share (ncu launches are
                cold-cache and serialised: compare SHARES with the bench, not absolute times)
full capture -> DRAM bytes, duration, achieved bandwidth, tensor-pipe activity, top stall reasons,
                hottest SASS instructions.
"""
import collections
import csv
import io
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0]
        if "gemm_tc_kernel" in d["Kernel Name"]:
            name = d["Kernel Name"].split("(")[0] + " grid=" + d.get("Grid Size", "")
        agg[name][0] += 1
        agg[name][1] += float(d["Metric Value"].replace(",", ""))
    tot = sum(v[1] for v in agg.values()) or 1.0
    out = io.StringIO()
    out.write(f"# ncu launch list: {sum(v[0] for v in agg.values())} launches, {tot / 1e3:.1f} us total\n")
    out.write(f"{'kernel':72s} {'n':>6s} {'total_us':>10s} {'avg_us':>8s} {'share':>6s}\n")
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.write(f"{k[:72]:72s} {n:6d} {t / 1e3:10.1f} {t / n / 1e3:8.2f} {100 * t / tot:5.1f}%\n")
    return out.getvalue()


def full(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "dram__bytes_read.sum.per_second", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "launch__grid_size",
            "launch__cluster_size", "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum"]
    out = io.StringIO()
    for r in rows[2:]:
        out.write(f"## {r[hdr.index('Kernel Name')][:110]}\n")
        for k in keys:
            if k in hdr:
                i = hdr.index(k)
                out.write(f"  {k} = {r[i]} {units[i]}\n")
        stalls = [(float(r[i]), h) for i, h in enumerate(hdr)
                  if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")
                  and r[i] not in ("", "n/a")]
        stalls.sort(reverse=True)
        out.write("  top stalls (warps per issue): " + ", ".join(
            f"{h.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}={v:.2f}"
            for v, h in stalls[:6]) + "\n")
    sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                          capture_output=True, text=True).stdout
    srows = list(csv.reader(io.StringIO(sass)))
    if len(srows) > 2:
        h = srows[1]
        if "Warp Stall Sampling (All Samples)" in h:
            i = h.index("Warp Stall Sampling (All Samples)")
            data = []
            for r in srows[2:]:
                try:
                    data.append((float(r[i]), r[1].strip()))
                except (ValueError, IndexError):
                    pass
            tot = sum(v for v, _ in data) or 1.0
            agg = collections.defaultdict(float)
            for v, s in data:
                agg[s] += v
            out.write("  hottest SASS (share of stall samples):\n")
            for s, v in sorted(agg.items(), key=lambda kv: -kv[1])[:12]:
                out.write(f"    {100 * v / tot:5.1f}%  {s[:90]}\n")
    return out.getvalue()


if __name__ == "__main__":
    tag = sys.argv[1]
    if len(sys.argv) > 2 and os.path.exists(sys.argv[2]):
        open(os.path.join(HERE, f"{tag}_launches.txt"), "w").write(launches(sys.argv[2]))
    if len(sys.argv) > 3 and os.path.exists(sys.argv[3]):
        open(os.path.join(HERE, f"{tag}_gemm_full.txt"), "w").write(full(sys.argv[3]))
