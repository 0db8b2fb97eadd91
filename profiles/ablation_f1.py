"""Table 1 ablation on one B200: the U-MLP (C4 shape) with the
three torchgpipe components switched on incrementally -- Fork/Join backward order, copy streams,
portals.  All partitions share cuda:0 (this round has one GPU), each on its own streams: the
numbers are directional, the paper's are four P40s.  Per row: training samples/s (median step),
device busy fraction (union of compute-task intervals over the step, from the trace), the
partitions' static memory plan, and copy payload bytes per step.

usage: python profiles/ablation_f1.py [--d 2048] [--batch 128] [--chunks 8] [--parts 4] [--steps 10]
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2004_09910_b200 import Pipeline, balance_by_time  # noqa: E402
from synth import configs as C  # noqa: E402

ROWS = [
    ("x x x", {"ablate_order": 11, "ablate_copy_streams": 1, "ablate_portals": 1}),
    ("Dependency x x", {"ablate_copy_streams": 1, "ablate_portals": 1}),
    ("Dependency Streams x", {"ablate_portals": 1}),
    ("Dependency Streams Portals", {}),
]


def busy_fraction(tl):
    """Union of compute-task intervals (stream 0) over [first start, last end]."""
    iv = sorted((int(a), int(b)) for p, s, k, i, a, b in tl if s == 0)
    if not iv:
        return 0.0
    tot, cur0, cur1 = 0, iv[0][0], iv[0][1]
    for a, b in iv[1:]:
        if a > cur1:
            tot += cur1 - cur0
            cur0, cur1 = a, b
        else:
            cur1 = max(cur1, b)
    tot += cur1 - cur0
    span = max(b for _, b in iv) - min(a for a, _ in iv)
    return tot / span


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--d", type=int, default=2048)
    ap.add_argument("--batch", type=int, default=128)
    ap.add_argument("--chunks", type=int, default=8)
    ap.add_argument("--parts", type=int, default=4)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--ckpt", default="except_last")
    a = ap.parse_args()
    layers = C.umlp(d=a.d)
    B = a.batch
    dev = torch.device("cuda", 0)
    X = torch.randn(B, a.d, device=dev)
    T = torch.randn(B, a.d, device=dev)
    Y = torch.empty_like(X)
    DY = torch.empty_like(X)
    bal, _ = balance_by_time(layers, a.parts, batch=B, chunks=a.chunks)  # torchgpipe.balance analog
    bal = [int(v) for v in bal]
    out = []
    base = None
    for name, opts in ROWS:
        P = Pipeline(layers, chunks=a.chunks, devices=[0] * a.parts, balance=bal, checkpoint=a.ckpt, max_batch=B, dtype="bf16",
                     seed=1)
        P.init_params(1)
        # F'/B pairing is this implementation's addition, not one of the paper's Table 1 components:
        # off in every arm so the rows compare the paper's design against its ablations
        P.set_option("pair_recompute", 0)
        for k, v in opts.items():
            P.set_option(k, v)

        def step():
            P.forward(X, B, Y)
            P.mse_loss_grad(Y, T, B, DY)
            P.backward(DY)
            P.step(0.01)

        for _ in range(3):
            step()
        ts = []
        b0, m0 = P.copy_stats()
        for _ in range(a.steps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            step()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        b1, m1 = P.copy_stats()
        P.set_trace(True)
        P.forward(X, B, Y)
        tf = P.timeline()
        P.mse_loss_grad(Y, T, B, DY)
        P.backward(DY)
        tb = P.timeline()
        P.step(0.01)
        P.set_trace(False)
        ms = statistics.median(ts)
        mem = sum(P.memory(j)["used"] for j in range(a.parts))
        row = dict(row=name, samples_per_s=round(B / ms * 1e3, 1), ms_per_step=round(ms, 3),
                   busy_fwd=round(busy_fraction(tf), 3), busy_bwd=round(busy_fraction(tb), 3),
                   plan_mem_gib=round(mem / 2**30, 3), copy_mb_per_step=round((b1 - b0) / a.steps / 1e6, 3),
                   messages_per_step=(m1 - m0) // a.steps)
        if base is None:
            base = row["samples_per_s"]
        row["speedup"] = round(row["samples_per_s"] / base, 3)
        out.append(row)
        print(json.dumps(row), flush=True)
        del P
    print(json.dumps({"config": dict(model=f"umlp d={a.d}", batch=B, chunks=a.chunks, parts=a.parts,
                                     devices="all on cuda:0", checkpoint=a.ckpt, balance=bal)}))


if __name__ == "__main__":
    main()
