"""Phase breakdown of the persistent forward-task kernel (run on the GPU box; sets TGP_PT_DEBUG):
for every grid barrier k, the time from the completion of barrier k-1 to (a) the first and (b) the
last CTA arrival and (c) the completion of k.  Barrier ids per block l: 3+5l GEMM1 partials, 4+5l
GEMM1 outputs, 5+5l GEMM2 partials, 6+5l GEMM2 outputs, 7+5l LN of the next block."""
import ctypes
import os
import sys

import numpy as np

os.environ.setdefault("TGP_PT_DEBUG", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2004_09910_b200 import Pipeline, tgp  # noqa: E402
from synth import configs as C  # noqa: E402

blocks = int(sys.argv[1]) if len(sys.argv) > 1 else 4
layers = C.resmlp_stack(blocks, 4096)
P = Pipeline(layers, chunks=32, devices=[0], balance=[blocks], checkpoint="never", max_batch=512, dtype="bf16", seed=1)
P.set_option("graphs", 0)
P.init_params(1)
X = torch.randn(512, 4096, device="cuda")
Y = torch.empty(512, 4096, device="cuda")
for _ in range(3):
    P.forward(X, 512, Y)
n = ctypes.c_int64()
L = tgp.lib()
L.tgp_debug_pt_read(P.h, 0, None, 0, ctypes.byref(n))
buf = np.zeros(n.value, dtype=np.uint64)
L.tgp_debug_pt_read(P.h, 0, buf.ctypes.data, n.value, ctypes.byref(n))
G = (n.value - 256) // (512 + 1024)
d = buf[:G * 512].reshape(G, 256, 2).astype(np.int64)
comp = buf[G * 512:G * 512 + 256].astype(np.int64)
ev = buf[G * 512 + 256:].reshape(G, 128, 8).astype(np.int64)
# per GEMM phase g: events relative to the completion of the barrier that made its B operand ready
evn = ["B first", "B last", "A last", "MMA first", "MMA done", "epi tfull", "epi last", "A first"]
print("GEMM phase events (median over CTAs, us after B-ready barrier; A issue times may be negative):")
for g in range(min(4, 2 * blocks)):
    need = (4 + 5 * (g >> 1)) if (g & 1) else (2 + 5 * (g >> 1))
    base = comp[need]
    vals = {evn[s]: np.median(ev[:, g, s] - base) / 1e3 for s in range(8) if (ev[:, g, s] > 0).all()}
    mx = {evn[s]: np.max(ev[:, g, s] - base) / 1e3 for s in range(8) if (ev[:, g, s] > 0).all()}
    print(f"  g={g}: " + "  ".join(f"{k} {v:6.2f} (max {mx[k]:6.2f})" for k, v in vals.items()))
nb = 1 + 5 * blocks
names = {0: "G1 partials", 1: "G1 out", 2: "G2 partials", 3: "G2 out", 4: "LN next"}
agg = {}
prev = comp[1]
for k in range(2, nb + 1):
    if comp[k] == 0:
        break
    arr = d[:, k, 0]
    nm = "LN x" if k == 2 else names[(k - 3) % 5]
    row = ((arr.min() - prev) / 1e3, (arr.max() - prev) / 1e3, (comp[k] - prev) / 1e3)
    agg.setdefault(nm, []).append(row)
    if k < 13:
        print(f"bar {k:3d} {nm:12s} first arrival +{row[0]:6.2f}  last arrival +{row[1]:6.2f}  complete +{row[2]:6.2f} us")
    prev = comp[k]
print("mean over blocks (us):")
for nm, rows in agg.items():
    r = np.mean(np.array(rows), axis=0)
    print(f"  {nm:12s} first {r[0]:6.2f}  last {r[1]:6.2f}  complete {r[2]:6.2f}")
tot = (prev - comp[1]) / 1e3
print(f"total {tot:.1f} us for {blocks} blocks -> {tot / blocks:.1f} us/block")
