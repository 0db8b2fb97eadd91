"""C4 (BASELINE configs[3]: U-MLP d = 2048, batch 256, m = 32, long skip routes) timed on one GPU:
n = 1 (one partition) and n = 8 partitions sharing the device (the multi-GPU code path; the
partitions' tasks overlap on separate streams, so this is NOT the 8-GPU number).
    python profiles/bench_c4.py [steps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2004_09910_b200 import Pipeline  # noqa: E402
from synth import configs as C  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
for n, bal in ((1, None), (8, [2, 3, 3, 3, 3, 3, 3, 3])):
    cfg = C.C4(n=n)
    P = Pipeline(cfg.layers, chunks=cfg.m, devices=[0] * n, balance=bal, checkpoint=cfg.checkpoint,
                 max_batch=cfg.batch, dtype="bf16", seed=1)
    P.init_params(1)
    d = cfg.layers[0]["d_in"]
    X = torch.randn(cfg.batch, d, device="cuda")
    T = torch.randn(cfg.batch, d, device="cuda")
    Y = torch.empty(cfg.batch, d, device="cuda")
    DY = torch.empty_like(Y)

    def step():
        P.forward(X, cfg.batch, Y)
        P.mse_loss_grad(Y, T, cfg.batch, DY)
        P.backward(DY)
        P.step(0.05)

    for _ in range(3):
        step()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(steps):
        step()
    b.record()
    b.synchronize()
    ms = a.elapsed_time(b) / steps
    print(f"C4 n={n} (one device): {ms:.2f} ms/step, {cfg.batch / ms * 1e3:.0f} samples/s, "
          f"{P.kernel_count()} kernels launched in total")
    P.close()
