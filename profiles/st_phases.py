"""Phase timeline of the persistent weight-streaming task kernel (run on the GPU box; sets
TGP_ST_DEBUG): per GEMM phase, the median / max over CTAs of each event relative to the phase's
first weight-tile issue, and the phase-to-phase period.
    python profiles/st_phases.py [blocks=4] [bwd=0] [nodep=0]"""
import ctypes
import os
import sys

import numpy as np

os.environ.setdefault("TGP_ST_DEBUG", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2004_09910_b200 import Pipeline, tgp  # noqa: E402
from synth import configs as C  # noqa: E402

opts = dict(a.split("=") for a in sys.argv[1:])
blocks = int(opts.get("blocks", 4))
bwd = int(opts.get("bwd", 0))
layers = C.resmlp_stack(blocks, 4096)
paired = int(opts.get("paired", 0))  # 1: stamps of the last PAIRED backward task (except_last, lane 1, half grid)
if paired:
    os.environ["TGP_ST_DEBUG"] = "2"
P = Pipeline(layers, chunks=32, devices=[0], balance=[blocks], checkpoint="except_last" if paired else "never",
             max_batch=512, dtype="bf16", seed=1)
P.set_option("stream_poll_ns", int(opts.get("poll", 32)))
P.set_option("stream_inflight", int(opts.get("inflight", 0)))
P.set_option("graphs", 0)
P.init_params(1)
X = torch.randn(512, 4096, device="cuda")
T = torch.randn(512, 4096, device="cuda")
Y = torch.empty(512, 4096, device="cuda")
DY = torch.empty_like(Y)
for _ in range(3):
    P.forward(X, 512, Y)
    if bwd:
        P.mse_loss_grad(Y, T, 512, DY)
        P.backward(DY)
n = ctypes.c_int64()
L = tgp.lib()
L.tgp_debug_stream_read(P.h, 0, None, 0, ctypes.byref(n))
buf = np.zeros(n.value, dtype=np.uint64)
L.tgp_debug_stream_read(P.h, 0, buf.ctypes.data, n.value, ctypes.byref(n))
NP = 2 * blocks
G = n.value // (NP * 13)
if paired:  # half grid: only the first G / 2 CTAs write
    G //= 2
    buf = buf[: G * NP * 13]
ev = buf.reshape(G, NP, 13).astype(np.int64)
names = ["B issue", "W first", "W last", "B landed", "MMA done", "TMEM rdy", "partials", "signal", "stats", "sig entry", "MMA half", "cp last", "bar passed"]
t0 = ev[:, 0, 1].min()
print(f"{'bwd' if bwd else 'fwd'} task, {blocks} blocks, {G} CTAs, ")
prev = None
for p in range(NP):
    base = np.median(ev[:, p, 1])
    row = []
    for s, nm in enumerate(names):
        v = ev[:, p, s]
        ok = v > 0
        if ok.sum() == 0:
            continue
        row.append(f"{nm} {(np.median(v[ok]) - base) / 1e3:6.2f}/{(np.max(v[ok]) - base) / 1e3:6.2f}")
    per = "" if prev is None else f"period {(base - prev) / 1e3:6.2f} us"
    prev = base
    print(f"p{p:2d} W-first@{(base - t0) / 1e3:8.2f} us {per} | " + " ".join(r.replace(' ', '=', 1) for r in row))
end = max(ev[:, :, 7].max(), ev[:, :, 4].max())
print(f"total {(end - t0) / 1e3:.1f} us -> {(end - t0) / 1e3 / NP:.2f} us per GEMM phase")
# per-CTA lag (which CTAs set the phase time): mean over phases of (MMA done - phase median), top 12
if int(opts.get("lag", 0)):
    lag = np.zeros(G)
    wl = np.zeros(G)
    for p in range(NP):
        v = ev[:, p, 4].astype(np.float64)
        w = ev[:, p, 2].astype(np.float64)
        ok = v > 0
        if ok.sum() < G // 2:
            continue
        lag += np.where(ok, v - np.median(v[ok]), 0.0)
        wl += np.where(w > 0, w - np.median(w[w > 0]), 0.0)
    lag /= NP
    wl /= NP
    order = np.argsort(-lag)
    print("CTA (cluster, rank): mean MMA-done lag us / mean last-weight-tile lag us")
    for cta in order[:12]:
        print(f"  cta {cta:3d} (cluster {cta // 4:2d}, rank {cta % 4}): {lag[cta] / 1e3:6.2f} / {wl[cta] / 1e3:6.2f}")
    print("lag by rank:", [round(float(lag[r::4].mean()) / 1e3, 2) for r in range(4)])
    print("lag by cluster (first 32):", [round(float(lag[4 * c:4 * c + 4].mean()) / 1e3, 1) for c in range(G // 4)])
