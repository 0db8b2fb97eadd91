"""Ad-hoc GPU diagnostic for the persistent forward task kernel (not collected by pytest)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from oracle import model as OM  # noqa: E402
from paper_2004_09910_b200 import Pipeline  # noqa: E402
from synth import configs as C  # noqa: E402
from synth import gen as G  # noqa: E402


def fwd(layers, x, params, pers, m):
    B = x.shape[0]
    P = Pipeline(layers, chunks=m, devices=[0], balance=[len(layers)], checkpoint="never", max_batch=B, dtype="bf16",
                 seed=3)
    P.set_option("persistent", pers)
    P.set_option("graphs", 0)
    for i, p in enumerate(params):
        P.set_param(i, p)
    X = torch.tensor(x, device="cuda")
    Y = torch.empty(B, layers[-1]["d_out"], device="cuda")
    P.forward(X, B, Y)
    y = Y.cpu().numpy()
    P.close()
    return y


for (nb, d, H) in [(1, 512, 512), (1, 2048, 2048), (1, 512, 1024), (2, 512, 512), (2, 2048, 4096)]:
    layers = C.resmlp_stack(nb, d, hidden=H)
    x, t = G.inputs(layers, 16, seed=5, dtype="bf16")
    params = G.params(layers, seed=5, dtype="bf16")
    ref, _ = OM.forward(layers, params, x)
    y0 = fwd(layers, x, params, 0, 1)
    y1 = fwd(layers, x, params, 1, 1)
    e0 = np.max(np.abs(y0 - ref)) / np.max(np.abs(ref))
    e1 = np.max(np.abs(y1 - ref)) / np.max(np.abs(ref))
    print(f"blocks={nb} d={d} H={H}: per-kernel err {e0:.2e}  persistent err {e1:.2e}  finite={np.isfinite(y1).all()}",
          flush=True)
    if e1 > 1e-2:
        diff = np.abs(y1 - ref)
        print("   rows max err", np.round(diff.max(axis=1) / np.max(np.abs(ref)), 3)[:16])
        print("   cols blocks (128) max err", np.round([diff[:, k:k + 128].max() for k in range(0, d, 128)], 3)[:16])
