"""F-task time of the stream kernel over runtime options (diagnostics).
    python profiles/st_sweep.py name=v1,v2,... [name2=...]   (each option swept alone, others default)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402,F401

from paper_2004_09910_b200 import Pipeline  # noqa: E402
from synth import configs as C  # noqa: E402

P = Pipeline(C.resmlp_stack(32, 4096), chunks=32, devices=[0], balance=[32], checkpoint="except_last", max_batch=512,
             dtype="bf16", seed=1)
P.init_params(1)
for arg in sys.argv[1:]:
    name, vals = arg.split("=")
    for v in vals.split(","):
        P.set_option(name, int(v))
        P.bench_dominant_gemm(0, 512, reps=2)
        ms, by, n = P.bench_dominant_gemm(0, 512, reps=10)
        print(f"{name}={v:>5s}: F task {ms * 1e3:7.1f} us = {ms * 1e3 / 64:5.2f} us/phase, {by / ms / 1e6:6.0f} GB/s",
              flush=True)
    P.set_option(name, 0)
