"""Small end-to-end cases for compute-sanitizer (memcheck / racecheck / synccheck): every kernel
family of the product path runs at least once -- the persistent stream kernel (F, paired F'/B,
fused sends), the fused W_j + SGD kernel, the per-layer tcgen05 GEMMs (U-MLP with portals), the
LayerNorm / Dropout kinds, fp32 SIMT, BatchNorm, and the GPT-2 kernels (attention, embedding, CE), and the asynchronous calls.
    compute-sanitizer --tool memcheck python profiles/diag/sanitize_case.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2004_09910_b200 import Pipeline  # noqa: E402
from synth import configs as C  # noqa: E402
from synth import gen as G  # noqa: E402


def run(layers, B, m, n, ckpt, dtype, fused=True, steps=2):
    P = Pipeline(layers, chunks=m, devices=[0] * n, checkpoint=ckpt, max_batch=B, dtype=dtype, seed=3)
    for i, p in enumerate(G.params(layers, seed=3, dtype=dtype)):
        P.set_param(i, p)
    x, t = G.inputs(layers, B if layers[0]["kind"] != "embed" else B // layers[0]["seq"], seed=3, dtype=dtype)
    X = torch.tensor(x, device="cuda")
    T = torch.tensor(t, device="cuda")
    Y = torch.empty(X.shape[0], layers[-1]["d_out"], device="cuda")
    DY = torch.empty_like(Y)
    for _ in range(steps):
        P.forward(X, X.shape[0], Y)
        loss = P.ce_loss_grad(Y, T, X.shape[0], DY) if layers[0]["kind"] == "embed" else P.mse_loss_grad(Y, T, X.shape[0], DY)
        if fused:
            P.backward_step(DY, 0.05)
        else:
            P.backward(DY)
            P.step(0.05)
    P.close()
    return loss


def run_async(layers, B, m, n):
    """the asynchronous stream-ordered calls (tgp_*_async + tgp_sync) on a side stream"""
    P = Pipeline(layers, chunks=m, devices=[0] * n, checkpoint="except_last", max_batch=B, dtype="bf16", seed=3)
    for i, p in enumerate(G.params(layers, seed=3, dtype="bf16")):
        P.set_param(i, p)
    x, t = G.inputs(layers, B, seed=3, dtype="bf16")
    X = torch.tensor(x, device="cuda")
    T = torch.tensor(t, device="cuda")
    Y = torch.empty(B, layers[-1]["d_out"], device="cuda")
    DY = torch.empty_like(Y)
    loss = torch.zeros(1, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    st = torch.cuda.Stream()
    for _ in range(2):
        P.forward_async(X, B, Y, stream=st)
        P.mse_loss_grad_async(Y, T, B, DY, loss, stream=st)
        P.backward_step_async(DY, 0.05, stream=st)
    P.sync()
    st.synchronize()
    P.close()
    return float(loss.item())


cases = [
    ("stream 2 partitions, pairing, fused send, W+SGD", lambda: run(C.resmlp_stack(4, 512, hidden=1024, dropout=0.1), 64, 4, 2, "except_last", "bf16")),
    ("U-MLP per-layer GEMMs + portals", lambda: run(C.umlp(d=256, levels=2, blocks_per_level=1, mid_blocks=1), 64, 2, 2, "always", "bf16")),
    ("LayerNorm / Dropout kinds bf16", lambda: run(C.ln_mlp(2, 256), 32, 2, 2, "except_last", "bf16", fused=False)),
    ("fp32 SIMT + BatchNorm", lambda: run(C.bn_mlp(4, 256), 64, 4, 2, "always", "fp32", fused=False)),
    ("stream 2 partitions, async ABI", lambda: run_async(C.resmlp_stack(4, 512, hidden=1024, dropout=0.1), 64, 4, 2)),
    ("GPT-2 tiny (attention, embedding, CE)", lambda: run(C.gpt2_stack(2, 128, 2, 128, 512, 0.1), 2 * 128, 2, 2, "always", "bf16", fused=False)),
]
only = sys.argv[1:] and [int(a) for a in sys.argv[1:]]
for k, (name, fn) in enumerate(cases):
    if only and k not in only:
        continue
    loss = fn()
    print(f"case {k} ({name}): loss {loss:.6f} finite {np.isfinite(loss)}", flush=True)
