"""Model-size scaling on B200 (the paper's Table 3 analog, PAPER.md P:312-317 /
P:339-349: "the model size scales linearly with the number of devices").

For each checkpoint mode, find the largest number of C2 blocks (pre-LN residual MLP, width 4096,
batch 512, m = 32, bf16 operands / fp32 master + grads) ONE B200 can hold as one pipeline partition:
a context is created with only that partition local and must leave 2 GiB free (the other partitions' devices = -1, nothing
allocated for them), so every device buffer of the static plan (parameters, gradients, bf16
shadow, dW operand stash, activation slots, receive arena, workspaces) is really allocated on the
GPU; a trial fails with TGP_E_NOMEM.  Partitions 0 and n-1 are checked (they hold the input / output
buffers).  Since each GPU holds one partition, the largest pipeline over n GPUs holds n times that
many blocks.  The n = 1 maximum is then trained for one step to show it is trainable.

    python profiles/mem_scaling.py
"""
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2004_09910_b200 import Pipeline  # noqa: E402
from paper_2004_09910_b200.tgp import TgpError  # noqa: E402
from synth import configs as C  # noqa: E402

D, B, M = 4096, 512, 32
HEADROOM = 2 << 30


def fits(blocks_per_part, n, part, mode):
    layers = C.resmlp_stack(blocks_per_part * n, D)
    devices = [-1] * n
    devices[part] = 0
    try:
        P = Pipeline(layers, chunks=M, devices=devices, balance=[blocks_per_part] * n, checkpoint=mode,
                     max_batch=B, dtype="bf16")
    except TgpError:
        torch.cuda.synchronize()
        return None
    mem = P.memory(part)
    free = torch.cuda.mem_get_info(0)[0]
    P.close()
    # headroom for what the static plan does not hold: CUDA graph instantiation of the task
    # sequences, the caller's x / y / dy / target tensors (4 x 8 MiB) and the CUDA context
    return mem if free >= HEADROOM else None


def max_blocks(mode, n=2):
    lo, hi = 1, 1
    while fits(hi, n, 0, mode) and fits(hi, n, n - 1, mode):
        lo, hi = hi, hi * 2
    while hi - lo > 1:
        mid = (lo + hi) // 2
        if fits(mid, n, 0, mode) and fits(mid, n, n - 1, mode):
            lo = mid
        else:
            hi = mid
    return lo, fits(lo, n, 0, mode)


out = {"workload": "C2 blocks (pre-LN residual MLP d 4096, batch 512, m 32, bf16 / fp32 master)",
       "device_total_gb": torch.cuda.mem_get_info(0)[1] / 1e9, "modes": {}}
params_per_block = 2 * D * D + 4 * D
for mode in ("never", "except_last", "always"):
    t0 = time.time()
    b, mem = max_blocks(mode)
    out["modes"][mode] = {
        "max_blocks_per_gpu": b, "plan_used_gb": mem["used"] / 1e9, "param_state_gb": mem["params"] / 1e9,
        "search_s": time.time() - t0,
        "max_params_billion": {str(n): round(n * b * params_per_block / 1e9, 1) for n in (1, 2, 4, 8)}}
    print(json.dumps({mode: out["modes"][mode]}), flush=True)

# the n = 1 maximum (checkpoint = always) trains
b = out["modes"]["always"]["max_blocks_per_gpu"]
layers = C.resmlp_stack(b, D)
P = Pipeline(layers, chunks=M, devices=[0], checkpoint="always", max_batch=B, dtype="bf16")
P.init_params(seed=1)
X = torch.randn(B, D, device="cuda")
T = torch.randn(B, D, device="cuda")
Y = torch.empty(B, D, device="cuda")
DY = torch.empty(B, D, device="cuda")
t0 = time.time()
P.forward(X, B, Y)
loss = P.mse_loss_grad(Y, T, B, DY)
P.backward(DY)
P.step(0.05)
torch.cuda.synchronize()
out["n1_max_step"] = {"blocks": b, "params_billion": round(b * params_per_block / 1e9, 2), "loss": loss,
                      "step_s": time.time() - t0}
print(json.dumps(out))
