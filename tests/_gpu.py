"""Helpers for the -m gpu parity tests: run one training step through the C ABI and compare with
the oracle on the same seeded inputs (synth/)."""
import numpy as np

from oracle import model as OM
from synth import configs as C
from synth import gen as G


def nwise_err(a, r, floor=0.0):
    a = np.asarray(a, np.float64).ravel()
    r = np.asarray(r, np.float64).ravel()
    den = max(np.max(np.abs(r)) if r.size else 0.0, floor, 1e-300)
    return float(np.max(np.abs(a - r)) / den) if r.size else 0.0


def gpu_step(layers, params, x, t, *, m, n, ckpt, dtype, lr, balance=None, seed=0, devices=None, options=None,
             steps=1, want_dx=True):
    import torch

    from paper_2004_09910_b200 import Pipeline

    B = x.shape[0]
    devices = devices or [0] * n
    P = Pipeline(layers, chunks=m, devices=devices, balance=balance, checkpoint=ckpt, max_batch=B, dtype=dtype,
                 seed=seed)
    for k, v in (options or {}).items():
        P.set_option(k, v)
    for idx, p in enumerate(params):
        P.set_param(idx, p)
    dev = torch.device("cuda", devices[0])
    X = torch.tensor(np.asarray(x, np.float32), device=dev)
    T = torch.tensor(np.asarray(t, np.float32), device=dev)
    d_out = layers[-1]["d_out"]
    Y = torch.empty(B, d_out, device=dev)
    DY = torch.empty(B, d_out, device=dev)
    DX = torch.empty(B, layers[0]["d_in"], device=dev)
    out = []
    for s in range(steps):
        P.forward(X, B, Y)
        loss = P.mse_loss_grad(Y, T, B, DY)
        P.backward(DY, DX if want_dx else None)
        grads = [P.get_grad(i) for i in range(P.n_params)]
        rec = dict(loss=loss, y=Y.cpu().numpy().astype(np.float64), dx=DX.cpu().numpy().astype(np.float64),
                   grads=grads, log=P.issue_log(), kernels=P.kernel_count())
        P.step(lr)
        rec["params"] = [P.get_param(i) for i in range(P.n_params)]
        out.append(rec)
    rec = out[-1] if steps == 1 else out
    return rec, P


def compare(gpu, ref, params, tol, lr, gpu_base=None):
    """Normwise per-tensor errors (reading Z15): loss (scalar relative), y, dx, every grad, every
    delta-theta = theta' - theta (GPU delta taken from `gpu_base` when given, e.g. after a first
    GPU step).  A gradient that is mathematically zero (e.g. the bias of a Linear feeding a
    BatchNorm, whose mean the BN removes) is compared against the fp32 round-off of the terms it
    sums: floor 1e-2 of the largest gradient instead of 1e-3."""
    errs = {}
    errs["loss"] = abs(gpu["loss"] - ref["loss"]) / abs(ref["loss"])
    errs["y"] = nwise_err(gpu["y"], ref["y"])
    errs["dx"] = nwise_err(gpu["dx"], ref["dx"])
    scale = max(np.max(np.abs(g)) for g in ref["grads"])
    for k, (g, gr) in enumerate(zip(gpu["grads"], ref["grads"])):
        zero = np.max(np.abs(gr)) <= 1e-9 * scale
        errs[f"g{k}"] = nwise_err(g, gr, (1e-2 if zero else 1e-3) * scale)
    base = gpu_base if gpu_base is not None else params
    for k, (pn, pr, p0, pb) in enumerate(zip(gpu["params"], ref["params"], params, base)):
        # delta-theta, allowing the fp32 rounding of the stored master weight theta' (|theta'| 2^-24
        # per element) that differencing two fp32 weights exposes when lr*g << theta
        pn = np.asarray(pn, np.float64).ravel()
        d_gpu = pn - np.asarray(pb, np.float64).ravel()
        d_ref = np.asarray(pr, np.float64).ravel() - np.asarray(p0, np.float64).ravel()
        excess = np.maximum(np.abs(d_gpu - d_ref) - 2.0 ** -24 * np.abs(pn), 0.0)
        zero = np.max(np.abs(d_ref)) <= 1e-9 * scale * lr
        den = max(np.max(np.abs(d_ref)), (1e-2 if zero else 1e-3) * scale * lr, 1e-300)
        errs[f"dtheta{k}"] = float(np.max(excess) / den)
    bad = {k: v for k, v in errs.items() if not (v <= tol)}
    return errs, bad


def oracle_step(layers, params, x, t, *, lr, m, seed=0, step=0):
    return OM.train_step(layers, params, x, t, lr=lr, m=m, seed=seed, step=step)


def bf16_shadow(layers, params):
    """The weights a bf16-mode GEMM reads after an SGD step (reading Z14: the bf16 shadow of the fp32
    master): weight matrices rounded to bf16, vectors (biases, LN gamma / beta) kept.  Applied to
    ORACLE parameters (e.g. the oracle's own step-0 result) to form the oracle's step-1 input, so the
    rounding of the inputs is not counted as error (O1) -- nothing here comes from the CUDA path."""
    out = []
    for (li, name, shape), p in zip(C.param_shapes(layers), params):
        p = np.asarray(p, np.float64)
        out.append(G.round_bf16(p).astype(np.float64) if len(shape) == 2 and name not in ("wte", "wpe") else p)
    return out


def make_case(layers, B, seed, dtype, x_mean=0.0, ln="default"):
    x, t = G.inputs(layers, B, seed=seed, dtype=dtype, x_mean=x_mean)
    params = G.params(layers, seed=seed, dtype=dtype, ln=ln)
    return x, t, params
