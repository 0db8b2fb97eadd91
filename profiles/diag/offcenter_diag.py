"""Diagnosis of off-centre parity: normwise errors of the stream kernel and the
per-layer path (stream off) against the fp64 oracle over two steps, x ~ N(mu, 1), wide LN params."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "..", "tests"))
import numpy as np

from _gpu import compare, gpu_step, make_case, oracle_step
from synth import configs as C
from synth import gen as G

for x_mean in [float(a) for a in (sys.argv[1:] or ["4", "32"])]:
    layers = C.resmlp_stack(4, 4096, dropout=0.1)
    B, m, lr, seed = 64, 4, 0.05, 31
    x, t, params = make_case(layers, B, seed, "bf16", x_mean=x_mean, ln="wide")
    ref0 = oracle_step(layers, params, x, t, lr=lr, m=m, seed=seed, step=0)
    ref1 = oracle_step(layers, ref0["params"], x, t, lr=lr, m=m, seed=seed, step=1)
    r1b = [G.round_bf16(p) for p in ref0["params"]]
    ref1b = oracle_step(layers, r1b, x, t, lr=lr, m=m, seed=seed, step=1)
    for stream in (1, 0):
        g, P = gpu_step(layers, params, x, t, m=m, n=1, ckpt="except_last", dtype="bf16", lr=lr, seed=seed,
                        steps=2, options={"stream": stream})
        P.close()
        e0, _ = compare(g[0], ref0, params, 2e-2, lr)
        e1, _ = compare(g[1], ref1, ref0["params"], 2e-2, lr, gpu_base=g[0]["params"])
        e1b, _ = compare(g[1], ref1b, r1b, 2e-2, lr, gpu_base=g[0]["params"])
        for name, e in (("step0", e0), ("step1", e1), ("step1_bf16w", e1b)):
            top = sorted(e.items(), key=lambda kv: -kv[1])[:6]
            print(f"mu={x_mean} stream={stream} {name}: " + " ".join(f"{k}={v:.2e}" for k, v in top), flush=True)
