"""Step breakdown of C2 at n = 1, m = 32 (run on the GPU box): per-task device times from the
CUDA-event task timeline, plus the forward / loss / backward / SGD calls timed with CUDA events.
    python profiles/step_breakdown.py [ckpt=except_last] [blocks=32] [option=value ...]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2004_09910_b200 import Pipeline  # noqa: E402
from synth import configs as C  # noqa: E402

opts = dict(a.split("=") for a in sys.argv[1:])
blocks = int(opts.pop("blocks", 32))
ckpt = opts.pop("ckpt", "except_last")
layers = C.resmlp_stack(blocks, 4096)
B, m = 512, 32
P = Pipeline(layers, chunks=m, devices=[0], balance=[blocks], checkpoint=ckpt, max_batch=B, dtype="bf16", seed=1)
for k, v in opts.items():
    P.set_option(k, int(v))
P.init_params(1)
X = torch.randn(B, 4096, device="cuda")
T = torch.randn(B, 4096, device="cuda")
Y = torch.empty(B, 4096, device="cuda")
DY = torch.empty_like(Y)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
calls = []
for it in range(5):
    if it == 4:
        P.set_trace(True)
    torch.cuda.synchronize()
    ev[0].record()
    P.forward(X, B, Y)
    ev[1].record()
    P.mse_loss_grad(Y, T, B, DY)
    ev[2].record()
    P.backward(DY)
    ev[3].record()
    if it < 4:
        P.step(1e-4)
    ev[4].record()
    torch.cuda.synchronize()
    calls.append([ev[k].elapsed_time(ev[k + 1]) for k in range(4)])
c = np.median(np.array(calls[1:4]), axis=0)
print(f"[{ckpt} {opts}] calls (ms): forward {c[0]:.2f}  loss {c[1]:.3f}  backward {c[2]:.2f}  step {c[3]:.2f}  "
      f"total {c.sum():.2f}")
tl = P.timeline()
names = {0: "F", 1: "F'", 2: "B", 7: "W"}
for k in (0, 1, 2, 7):
    d = [(r[5] - r[4]) / 1e3 for r in tl if int(r[1]) == 0 and int(r[2]) == k]
    if d:
        print(f"  {names[k]:2s} n={len(d):3d} mean {np.mean(d):9.1f} us  min {np.min(d):9.1f}  max {np.max(d):9.1f}"
              f"  sum {np.sum(d) / 1e3:7.2f} ms")
P.close()
