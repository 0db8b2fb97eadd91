"""GPU tests of the asynchronous, stream-ordered ABI (tgp_*_async + tgp_sync; include/tgp.h;
SURVEY 8(f) f3; PAPER.md P:133 / Alg. 1: the host only issues, the devices wait).

An async call issues exactly the device work of its blocking twin, so a training run driven through
the async calls must be BITWISE equal to the same run through the blocking calls -- with the inputs
still in production on the caller's stream when the call is issued (a device sleep, then the copy
that writes x / dy, both queued before the call): a call that did not order itself after the
caller's stream would read stale inputs.  A second test checks the call really returns before its
device work ends, and a third checks the result against the fp64 oracle."""
import time

import numpy as np
import pytest

from synth import configs as C

from _gpu import compare, make_case, oracle_step

pytestmark = pytest.mark.gpu

SLEEP = 20_000_000  # ~10 ms of device cycles queued ahead of every input copy


def _blocking(layers, params, x, t, *, m, n, ckpt, dtype, lrs, fused, seed=3):
    import torch

    from paper_2004_09910_b200 import Pipeline

    B = x.shape[0]
    P = Pipeline(layers, chunks=m, devices=[0] * n, checkpoint=ckpt, max_batch=B, dtype=dtype, seed=seed)
    for i, p in enumerate(params):
        P.set_param(i, p)
    X = torch.tensor(np.asarray(x, np.float32), device="cuda")
    T = torch.tensor(np.asarray(t, np.float32), device="cuda")
    Y = torch.empty(B, layers[-1]["d_out"], device="cuda")
    DY = torch.empty_like(Y)
    DX = torch.empty(B, layers[0]["d_in"], device="cuda")
    losses = []
    for lr in lrs:
        P.forward(X, B, Y)
        losses.append(P.mse_loss_grad(Y, T, B, DY))
        if fused:
            P.backward_step(DY, lr, DX)
        else:
            P.backward(DY, DX)
            P.step(lr)
    out = dict(losses=losses, params=[P.get_param(i) for i in range(P.n_params)], dx=DX.cpu().numpy(),
               y=Y.cpu().numpy())
    P.close()
    return out


def _async(layers, params, x, t, *, m, n, ckpt, dtype, lrs, fused, seed=3):
    """Same run through the async calls on a side stream; x and the target are (re)written on that
    stream after a device sleep right before each forward, and nothing waits on the host until the end."""
    import torch

    from paper_2004_09910_b200 import Pipeline

    B = x.shape[0]
    P = Pipeline(layers, chunks=m, devices=[0] * n, checkpoint=ckpt, max_batch=B, dtype=dtype, seed=seed)
    for i, p in enumerate(params):
        P.set_param(i, p)
    st = torch.cuda.Stream()
    Xh = torch.tensor(np.asarray(x, np.float32)).pin_memory()
    Th = torch.tensor(np.asarray(t, np.float32)).pin_memory()
    X = torch.zeros(B, layers[0]["d_in"], device="cuda")
    T = torch.zeros(B, layers[-1]["d_out"], device="cuda")
    Y = torch.empty(B, layers[-1]["d_out"], device="cuda")
    DY = torch.empty_like(Y)
    DX = torch.empty(B, layers[0]["d_in"], device="cuda")
    loss = torch.zeros(len(lrs), dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    with torch.cuda.stream(st):
        for k, lr in enumerate(lrs):
            X.zero_()
            T.zero_()
            torch.cuda._sleep(SLEEP)
            X.copy_(Xh, non_blocking=True)
            T.copy_(Th, non_blocking=True)
            P.forward_async(X, B, Y, stream=st)
            P.mse_loss_grad_async(Y, T, B, DY, loss[k:k + 1], stream=st)
            if fused:
                P.backward_step_async(DY, lr, DX, stream=st)
            else:
                P.backward_async(DY, DX, stream=st)
                P.step_async(lr, stream=st)
    P.sync()
    st.synchronize()
    out = dict(losses=[float(v) for v in loss.cpu().numpy()], params=[P.get_param(i) for i in range(P.n_params)],
               dx=DX.cpu().numpy(), y=Y.cpu().numpy())
    P.close()
    return out


def _same(a, b):
    assert a["losses"] == b["losses"]
    assert np.array_equal(a["y"], b["y"])
    assert np.array_equal(a["dx"], b["dx"])
    for k, (pa, pb) in enumerate(zip(a["params"], b["params"])):
        assert np.array_equal(pa, pb), k


@pytest.mark.parametrize("fused", [False, True])
def test_async_bitwise_equals_blocking_stream_kernel(fused):
    # 2 partitions of RESMLP blocks (persistent stream kernel, fused sends, F'/B pairing), dropout
    layers = C.resmlp_stack(4, 512, hidden=1024, dropout=0.1)
    x, t, params = make_case(layers, 64, 11, "bf16")
    kw = dict(m=4, n=2, ckpt="except_last", dtype="bf16", lrs=[0.05, 0.05, 0.02], fused=fused)
    _same(_blocking(layers, params, x, t, **kw), _async(layers, params, x, t, **kw))


def test_async_bitwise_equals_blocking_per_layer_fp32():
    # fp32 per-layer kernels and push-kernel copies between 3 partitions (no stream kernel)
    layers = C.mlp_chain(6, 64)
    x, t, params = make_case(layers, 24, 12, "fp32")
    kw = dict(m=4, n=3, ckpt="always", dtype="fp32", lrs=[0.1, 0.1], fused=False)
    _same(_blocking(layers, params, x, t, **kw), _async(layers, params, x, t, **kw))


def test_async_call_returns_before_its_work_and_matches_oracle():
    import torch

    from paper_2004_09910_b200 import Pipeline

    layers = C.resmlp_stack(4, 512, hidden=1024)
    B, m, lr = 64, 4, 0.05
    x, t, params = make_case(layers, B, 13, "bf16")
    P = Pipeline(layers, chunks=m, devices=[0, 0], checkpoint="except_last", max_batch=B, dtype="bf16", seed=0)
    for i, p in enumerate(params):
        P.set_param(i, p)
    X = torch.tensor(np.asarray(x, np.float32), device="cuda")
    T = torch.tensor(np.asarray(t, np.float32), device="cuda")
    Y = torch.empty(B, layers[-1]["d_out"], device="cuda")
    DY = torch.empty_like(Y)
    DX = torch.empty(B, layers[0]["d_in"], device="cuda")
    # warm-up through the blocking calls (descriptors for this B, task graphs captured), then the
    # weights restored and the gradients reset (a step with lr = 0), so the async step starts clean
    P.forward(X, B, Y)
    P.mse_loss_grad(Y, T, B, DY)
    P.backward(DY, DX)
    P.step(0.0)
    for i, p in enumerate(params):
        P.set_param(i, p)
    st = torch.cuda.Stream()
    loss = torch.zeros(1, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    with torch.cuda.stream(st):
        torch.cuda._sleep(SLEEP * 20)  # ~200 ms on the caller's stream
        t0 = time.perf_counter()
        P.forward_async(X, B, Y, stream=st)
        P.mse_loss_grad_async(Y, T, B, DY, loss, stream=st)
        P.backward_async(DY, DX, stream=st)
        issue_s = time.perf_counter() - t0
        busy = not st.query()
    P.sync()
    st.synchronize()
    grads = [P.get_grad(i) for i in range(P.n_params)]
    P.step(lr)
    gpu = dict(loss=float(loss.item()), y=Y.cpu().numpy().astype(np.float64), dx=DX.cpu().numpy().astype(np.float64),
               grads=grads, params=[P.get_param(i) for i in range(P.n_params)])
    P.close()
    assert busy, "the caller's stream finished before the async calls returned"
    assert issue_s < 0.1, issue_s  # the calls did not wait for the ~200 ms sleep queued before them
    ref = oracle_step(layers, params, x, t, m=m, lr=lr, seed=0)
    errs, bad = compare(gpu, ref, params, 2e-2, lr)
    assert not bad, bad
