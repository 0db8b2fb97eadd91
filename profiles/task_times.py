"""Per-task device times (CUDA-event task timeline) of one C2 training step at n = 1, m = 32, under
runtime options given as key=value arguments (e.g. persistent=0).  Run on the GPU box."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2004_09910_b200 import Pipeline  # noqa: E402
from synth import configs as C  # noqa: E402

opts = dict(a.split("=") for a in sys.argv[1:])
blocks = int(opts.pop("blocks", 32))
layers = C.resmlp_stack(blocks, 4096)
B, m = 512, 32
P = Pipeline(layers, chunks=m, devices=[0], balance=[blocks], checkpoint="except_last", max_batch=B, dtype="bf16",
             seed=1)
for k, v in opts.items():
    P.set_option(k, int(v))
P.init_params(1)
X = torch.randn(B, 4096, device="cuda")
T = torch.randn(B, 4096, device="cuda")
Y = torch.empty(B, 4096, device="cuda")
DY = torch.empty_like(Y)
for it in range(3):
    if it == 2:
        P.set_trace(True)
    P.forward(X, B, Y)
    P.mse_loss_grad(Y, T, B, DY)
    P.backward(DY)
    if it < 2:
        P.step(1e-4)
tl = P.timeline()
names = {0: "F", 1: "F'", 2: "B", 7: "W"}
for k in (0, 1, 2, 7):
    d = [(r[5] - r[4]) / 1e3 for r in tl if int(r[1]) == 0 and int(r[2]) == k]
    if d:
        print(f"{names[k]:2s} n={len(d):3d} mean {np.mean(d):9.1f} us  min {np.min(d):9.1f}  max {np.max(d):9.1f}")
fw = [r for r in tl if int(r[2]) in (0,)]
bw = [r for r in tl if int(r[2]) in (1, 2, 7)]
print(f"forward call span {(max(r[5] for r in fw) - min(r[4] for r in fw)) / 1e3:.1f} us, "
      f"backward span {(max(r[5] for r in bw) - min(r[4] for r in bw)) / 1e3:.1f} us")
