"""Full-size C2 (32 x 4096, B = 512, m = 32): checkpoint modes must give bitwise-identical loss and
gradients (F' == F, reading Z21).  Prints the first mismatching parameter, if any."""
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
B = 512
g = torch.Generator().manual_seed(5)
X = torch.randn(B, 4096, generator=g).cuda()
T = torch.randn(B, 4096, generator=g).cuda()
res = {}
for mode in ("except_last", "never", "always"):
    P = Pipeline(layers, chunks=32, devices=[0], balance=[blocks], checkpoint=mode, max_batch=B, dtype="bf16", seed=1)
    for k, v in opts.items():
        P.set_option(k, int(v))
    P.init_params(1)
    Y = torch.empty(B, 4096, device="cuda")
    DY = torch.empty_like(Y)
    losses = []
    for it in range(3):
        P.forward(X, B, Y)
        losses.append(P.mse_loss_grad(Y, T, B, DY))
        P.backward(DY)
        if it < 2:
            P.step(0.05)
    grads = [P.get_grad(i) for i in range(0, P.n_params, 7)]
    res[mode] = (losses, grads)
    P.close()
    print(mode, losses, flush=True)
for mode in ("never", "always"):
    same_l = res[mode][0] == res["except_last"][0]
    bad = [k for k, (a, b) in enumerate(zip(res[mode][1], res["except_last"][1])) if not np.array_equal(a, b)]
    print(f"{mode} vs except_last: losses equal {same_l}, grads mismatching (sampled idx) {bad[:10]}")
