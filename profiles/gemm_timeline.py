"""Per-CTA %globaltimer timeline of the dominant GEMM chain (needs the TGP_GEMM_TIMING variant:
TGP_LIB=variants/timing/libtgp.so, built by
profiles/build_variant.py timing -DTGP_GEMM_TIMING).  Prints, per launch of the chain, when its CTAs start,
pass griddepcontrol.wait, finish their MMAs, and exit -- relative to the previous launch's exit."""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402,F401

from paper_2004_09910_b200 import Pipeline, tgp  # noqa: E402
from synth import configs as C  # noqa: E402

sk = int(sys.argv[1]) if len(sys.argv) > 1 else 4
chunks = int(os.environ.get("CHUNKS", "32"))  # 32: 16-row micro-batches (stream kernel off below)
layers = C.resmlp_stack(32, 4096)
P = Pipeline(layers, chunks=chunks, devices=[0], balance=[32], checkpoint="except_last", max_batch=512, dtype="bf16",
             seed=1)
P.init_params(1)
P.set_option("splitk", sk)
P.set_option("stream", 0)
if "PF" in os.environ:
    P.set_option("prefetch", int(os.environ["PF"]))
lib = tgp.lib()
f = lib.tgp_debug_timestamps
f.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
f.restype = ctypes.c_int
P.bench_dominant_gemm(0, 512, reps=1)  # warm
buf = np.zeros((8192, 12), dtype=np.uint64)
f(buf.ctypes.data, 8192, 1)
ms, by, n = P.bench_dominant_gemm(0, 512, reps=1)
cnt = f(buf.ctypes.data, 8192, 1)
ncta = 32 * sk
rows = buf[:cnt].astype(np.int64)
own = rows[:, 6] > 0
for a_, b_, nm in ((3, 6, "tfull->recv"), (6, 8, "recv->sum"), (8, 9, "sum->epi_done"), (9, 7, "epi_done->stores"),
                   (7, 4, "stores->exit"), ):
    if not own.any() or rows[own, b_].min() == 0:
        continue
    d = rows[own, b_] - rows[own, a_]
    if False:
        continue
    print(f"{nm:18s} ns pct0/50/90/100", np.percentile(d, [0, 50, 90, 100]))
if len(sys.argv) > 2:
    np.save(sys.argv[2], rows)
# drop the warm-up round (first 32 launches) recorded in this window
launches = cnt // ncta
print(f"splitk={sk} chain avg {ms * 1e3:.2f} us/launch, {launches} launches recorded, {ncta} CTAs each")
t0 = rows[:, 0].min()
prev_end = None
for k in range(launches):
    r = rows[k * ncta:(k + 1) * ncta] - t0
    st, wt, mm, tf, en = r[:, 0], r[:, 1], r[:, 2], r[:, 3], r[:, 4]
    wt = wt[wt > -t0 // 2]
    raw = rows[k * ncta:(k + 1) * ncta]
    pu, rv, cs = (raw[:, c][raw[:, c] > 0] - t0 for c in (5, 6, 7))
    line = (f"L{k:02d} start[min {st.min() / 1e3:8.2f} max {st.max() / 1e3:8.2f}] "
            f"wait_done[min {wt.min() / 1e3:8.2f} max {wt.max() / 1e3:8.2f}] mma_done max {mm.max() / 1e3:8.2f} "
            f"epi_start max {tf.max() / 1e3:8.2f} exit[min {en.min() / 1e3:8.2f} max {en.max() / 1e3:8.2f}]")
    if len(pu) and len(rv) and len(cs):
        line += (f" push_done max {pu.max() / 1e3:8.2f} recv_done[min {rv.min() / 1e3:8.2f} max {rv.max() / 1e3:8.2f}]"
                 f" stores_done max {cs.max() / 1e3:8.2f}")
    if prev_end is not None:
        line += f"  dt(exit-exit) {(en.max() - prev_end) / 1e3:6.2f}"
    prev_end = en.max()
    print(line)
    if k > 12:
        break
