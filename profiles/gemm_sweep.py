"""GEMM-chain micro-sweep (run on the GPU box): average per-launch time of the dominant forward GEMM
of the C2 stack (32 layers, cold weights, PDL-chained like a task) under runtime options."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402,F401

from paper_2004_09910_b200 import Pipeline  # noqa: E402
from synth import configs as C  # noqa: E402

layers = C.resmlp_stack(32, 4096)
P = Pipeline(layers, chunks=32, devices=[0], balance=[32], checkpoint="except_last", max_batch=512, dtype="bf16",
             seed=1)
P.init_params(1)
res = {}
for pf in (0, 1):
    for sk in (2, 4, 8):
        for pdl in (0, 1):
            P.set_option("prefetch", pf)
            P.set_option("splitk", sk)
            P.set_option("pdl", pdl)
            ms, by, n = P.bench_dominant_gemm(0, 512, reps=3)
            key = f"prefetch={pf} splitk={sk} pdl={pdl}"
            res[key] = (round(ms * 1e3, 2), round(by / (ms * 1e-3) / 1e9, 1))
            print(key, "us/launch", res[key][0], "GB/s", res[key][1], flush=True)
json.dump(res, open(sys.argv[1] if len(sys.argv) > 1 else "gemm_sweep.json", "w"), indent=1)
