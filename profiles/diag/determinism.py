"""Diagnostics: is the stream-kernel forward / backward bitwise deterministic across repeated calls?
    python profiles/diag/determinism.py d L B m"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2004_09910_b200 import Pipeline  # noqa: E402
from synth import configs as C  # noqa: E402

d, L, B, m = (int(a) for a in sys.argv[1:5])
mode = sys.argv[5] if len(sys.argv) > 5 else "fb"    # fb: forward + backward per rep; f: forward only
pair = int(sys.argv[6]) if len(sys.argv) > 6 else 1
P = Pipeline(C.resmlp_stack(L, d), chunks=m, devices=[0], checkpoint="except_last", max_batch=B, dtype="bf16", seed=1)
P.init_params(1)
if pair >= 0:
    P.set_option("pair_recompute", pair)
for kv in sys.argv[7:]:
    k, v = kv.split("=")
    P.set_option(k, int(v))
g = torch.Generator(device="cpu").manual_seed(3)
X = torch.randn(B, d, generator=g).cuda()
T = torch.randn(B, d, generator=g).cuda()
Y = torch.empty(B, d, device="cuda")
DY = torch.empty_like(Y)
DX = torch.empty_like(Y)
ys, dxs = [], []
for r in range(4):
    P.forward(X, B, Y)
    if mode == "fb":
        P.mse_loss_grad(Y, T, B, DY)
        P.backward(DY, DX)
    ys.append(Y.cpu().numpy().copy())
    dxs.append(DX.cpu().numpy().copy())
for r in range(1, 4):
    dy = np.abs(ys[r] - ys[0])
    dd = np.abs(dxs[r] - dxs[0])
    rows = np.nonzero(dy.max(axis=1))[0]
    print(f"{mode} pair={pair} {sys.argv[7:]} d={d} L={L} B={B} m={m} rep {r}: y diff max {dy.max():.3e} rows {rows[:20].tolist()} ({len(rows)}), "
          f"dx diff max {dd.max():.3e} rows {len(np.nonzero(dd.max(axis=1))[0])}", flush=True)
