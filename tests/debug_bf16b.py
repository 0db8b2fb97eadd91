"""Ad-hoc GPU diagnostic (not collected by pytest)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch  # noqa: E402

from _gpu import compare, gpu_step, make_case, oracle_step  # noqa: E402
from synth import configs as C  # noqa: E402
from synth.gen import round_bf16  # noqa: E402
from paper_2004_09910_b200.tgp import test_gemm_bf16  # noqa: E402


def gemm(M, N, K, a_mn, splits):
    rs = np.random.default_rng(0)
    A = round_bf16(rs.standard_normal((M, K)).astype(np.float32))
    Bm = round_bf16(rs.standard_normal((N, K)).astype(np.float32))
    ref = A.astype(np.float64) @ Bm.astype(np.float64).T
    dA = torch.tensor(A.T.copy() if a_mn else A, device="cuda").to(torch.bfloat16)
    dB = torch.tensor(Bm, device="cuda").to(torch.bfloat16)
    D = torch.full((M * N,), float("nan"), device="cuda")
    test_gemm_bf16(dA, dB, D, M, N, K, a_mn, 0, splits)
    d = D.cpu().numpy().reshape(N, M).T
    return np.max(np.abs(d - ref)) / np.max(np.abs(ref))


for (M, N, K) in [(256, 16, 512), (512, 16, 256), (128, 16, 128), (256, 16, 256), (512, 16, 512)]:
    for a_mn in (0, 1):
        print(M, N, K, "a_mn", a_mn, [f"{gemm(M, N, K, a_mn, s):.2e}" for s in (1, 2, 4, 8)], flush=True)

for d, H in [(256, 512), (256, 256), (512, 512)]:
    layers = C.resmlp_stack(1, d, hidden=H)
    x, t, params = make_case(layers, 16, 7, "bf16")
    ref = oracle_step(layers, params, x, t, lr=0.05, m=1, seed=7)
    for sk in (1, 2, 4, 8):
        g, P = gpu_step(layers, params, x, t, m=1, n=1, ckpt="never", dtype="bf16", lr=0.05, seed=7,
                        options={"splitk": sk, "graphs": 0, "pdl": 0})
        errs, bad = compare(g, ref, params, 2e-2, 0.05)
        print(f"pipeline d={d} H={H} splitk={sk}: y={errs['y']:.2e} dx={errs['dx']:.2e} worst={max(errs.values()):.2e}",
              flush=True)
        P.close()
