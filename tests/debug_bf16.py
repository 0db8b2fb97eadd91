"""Ad-hoc GPU diagnostic (not collected by pytest): isolates bf16-path discrepancies."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

from _gpu import compare, gpu_step, make_case, oracle_step  # noqa: E402
from synth import configs as C  # noqa: E402


def run(layers, B, m, n, ckpt, dtype, opts):
    x, t, params = make_case(layers, B, 7, dtype)
    ref = oracle_step(layers, params, x, t, lr=0.05, m=m, seed=7)
    g, P = gpu_step(layers, params, x, t, m=m, n=n, ckpt=ckpt, dtype=dtype, lr=0.05, seed=7, options=opts)
    errs, bad = compare(g, ref, params, 2e-2, 0.05)
    worst = sorted(errs.items(), key=lambda kv: -kv[1])[:4]
    P.close()
    return errs["y"], errs["loss"], worst


if __name__ == "__main__":
    for d, H in [(128, 128), (256, 512)]:
        layers = C.resmlp_stack(1, d, hidden=H)
        for (m, n) in [(1, 1), (2, 1), (4, 1)]:
            for opts in [{"graphs": 0, "pdl": 0}, {"graphs": 0, "pdl": 1}, {"graphs": 1, "pdl": 0}, {"graphs": 1, "pdl": 1}]:
                B = 16 * m
                try:
                    ey, el, worst = run(layers, B, m, n, "never", "bf16", opts)
                    print(f"d={d} H={H} m={m} n={n} {opts}: y={ey:.3e} loss={el:.3e} worst={worst}", flush=True)
                except Exception as e:
                    print(f"d={d} m={m} n={n} {opts}: EXC {e}", flush=True)
    layers = [C.layer("linear", 128, 128, act="gelu"), C.layer("linear", 128, 256, act="none")]
    for (m, n) in [(1, 1), (2, 2)]:
        ey, el, worst = run(layers, 16 * m, m, n, "never", "bf16", {"graphs": 0, "pdl": 0})
        print(f"linear m={m} n={n}: y={ey:.3e} loss={el:.3e} worst={worst}", flush=True)
