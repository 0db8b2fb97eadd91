"""Task timeline -> Chrome Trace Event JSON (SPEC S:283 format; Fig. 7: blue = compute,
red = copy per device), and the per-device compute-order projection used by the order checker.

Rows come from Pipeline.timeline() after tgp_set_trace(1): (part, stream, kind, i, t0_ns, t1_ns),
stream 0 = compute, 1 = activation/gradient copies, 2 = skip copies; times are CUDA-event based,
relative to the start of the call on that partition's device.
"""
import json

KIND = {0: "F", 1: "F'", 2: "B", 3: "COPY_F", 4: "COPY_B", 5: "SKIP_F", 6: "SKIP_B", 7: "W"}


def chrome_trace(rows, offset_us=0.0):
    ev = []
    for part, stream, kind, i, t0, t1 in rows:
        ev.append({"name": f"{KIND[int(kind)]}{int(i)},{int(part) + 1}" if kind != 7 else f"W{int(part) + 1}",
                   "ph": "X", "ts": offset_us + t0 / 1e3, "dur": max(0.0, (t1 - t0) / 1e3), "pid": int(part),
                   "tid": int(stream), "args": {"task": KIND[int(kind)], "i": int(i), "j": int(part) + 1}})
    return ev


def write_chrome_trace(path, rows_fwd, rows_bwd=None):
    """Forward and backward calls have separate time origins; the backward is shifted after the
    forward's last event for display."""
    ev = chrome_trace(rows_fwd)
    if rows_bwd is not None and len(rows_bwd):
        end = max((e["ts"] + e["dur"] for e in ev), default=0.0)
        ev += chrome_trace(rows_bwd, offset_us=end + 10.0)
    with open(path, "w") as f:
        json.dump({"traceEvents": ev, "displayTimeUnit": "ns"}, f)
    return ev


def device_compute_order(rows):
    """Per partition, the compute tasks (kind, i) ordered by start time (order checker O11)."""
    out = {}
    for part, stream, kind, i, t0, t1 in sorted(rows, key=lambda r: (r[0], r[4])):
        if int(stream) == 0:
            out.setdefault(int(part), []).append((int(kind), int(i)))
    return out
