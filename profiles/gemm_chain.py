"""Runs the dominant GEMM chain (tgp_bench_dominant_gemm, C2 W1 GEMMs) a few rounds -- a small
target for `ncu -k regex:gemm_tc_kernel` source-level stall sampling."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402,F401

from paper_2004_09910_b200 import Pipeline  # noqa: E402
from synth import configs as C  # noqa: E402

sk = int(sys.argv[1]) if len(sys.argv) > 1 else 0
P = Pipeline(C.resmlp_stack(32, 4096), chunks=32, devices=[0], balance=[32], checkpoint="except_last", max_batch=512,
             dtype="bf16", seed=1)
P.init_params(1)
if sk:
    P.set_option("splitk", sk)
for kv in sys.argv[2:]:
    k, v = kv.split("=")
    P.set_option(k, int(v))
for _ in range(3):
    ms, by, n = P.bench_dominant_gemm(0, 512, reps=2)
print(f"{ms * 1e3:.2f} us/launch, {by / ms / 1e6:.0f} GB/s")
