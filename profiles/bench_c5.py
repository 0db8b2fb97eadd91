"""C5 timing (BASELINE.json configs[4]: GPT-2-1.5B-shaped stack, 48 blocks, d 1600, 25 heads, seq
1024, dropout 0.1, m = 32 micro-batches of one sequence, checkpoint = always) on ONE B200.

    python profiles/bench_c5.py [--layers 48] [--seqs 32] [--chunks 32] [--parts 1] [--steps 3]

All partitions share cuda:0 (this pool has one GPU per call), so this is the per-GPU work of the
pipeline run serially, not the 8-GPU number.  A step = forward + CE + backward (F' recompute under
the restored Philox counters) + SGD; timed with CUDA events around whole steps after warm-up (the
library calls are blocking).  Algorithmic FLOPs per token: 2 x matmul params + causal attention
2 seq d per layer (S and PV over seq/2 keys on average), x3 for training, +1x forward for recompute.
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2004_09910_b200 import Pipeline  # noqa: E402
from synth import configs as C  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--layers", type=int, default=48)
ap.add_argument("--seqs", type=int, default=32)
ap.add_argument("--chunks", type=int, default=32)
ap.add_argument("--parts", type=int, default=1)
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--warmup", type=int, default=2)
ap.add_argument("--checkpoint", default="always")
ap.add_argument("--dropout", type=float, default=0.1)
a = ap.parse_args()

layers = C.gpt2_stack(a.layers, dropout=a.dropout)
seq, V, d = layers[1]["seq"], layers[-1]["d_out"], layers[1]["d_in"]
T = a.seqs * seq
free0 = torch.cuda.mem_get_info(0)[0]
t0 = time.time()
P = Pipeline(layers, chunks=a.chunks, devices=[0] * a.parts, checkpoint=a.checkpoint, max_batch=T, dtype="bf16",
             seed=1)
P.init_params(seed=1)
create_s = time.time() - t0
free1 = torch.cuda.mem_get_info(0)[0]
g = torch.Generator(device="cuda").manual_seed(0)
X = torch.randint(0, V, (T, 1), device="cuda", generator=g).float()
Tg = torch.randint(0, V, (T,), device="cuda", generator=g).int()
Y = torch.empty(T, V, device="cuda")
DY = torch.empty(T, V, device="cuda")


def step():
    P.forward(X, T, Y)
    loss = P.ce_loss_grad(Y, Tg, T, DY)
    P.backward(DY)
    P.step(0.01)
    return loss


losses = [step() for _ in range(a.warmup)]
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
k0 = P.kernel_count()
e0.record()
for _ in range(a.steps):
    losses.append(step())
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.steps
n_mm = sum(12 * d * d + 0 for L in layers if L["kind"] == "transformer") + d * V  # Wqkv 3d^2, Wo d^2, W1/W2 8d^2
attn = sum(2 * seq * d for L in layers if L["kind"] == "transformer")
fwd = 2 * n_mm + attn
mult = 4 if a.checkpoint == "always" else 3
flops = fwd * mult * T
out = dict(workload=f"C5: embed + {a.layers} x GPT-2 block (d {d}, 25 heads, seq {seq}, dropout {a.dropout}) + LM head V {V}",
           seqs=a.seqs, chunks=a.chunks, parts_on_one_gpu=a.parts, checkpoint=a.checkpoint,
           ms_per_step=ms, seq_per_s=a.seqs / ms * 1e3, tokens_per_s=T / ms * 1e3,
           model_tflops=flops / ms * 1e-9, algorithmic_flop_per_step=flops,
           kernels_per_step=(P.kernel_count() - k0) / a.steps, create_s=create_s,
           memory_gb=(free0 - free1) / 1e9, loss_first_last=[losses[0], losses[-1]])
print(json.dumps(out))
