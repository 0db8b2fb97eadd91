"""GPU tests of tgp_backward_step: the deferred weight-gradient task W_j with the plain SGD update
fused into its epilogue (csrc/gemm_dw_sgd.cu; PAPER.md P:70 g^j = sum_i g_i^j, P:307 plain SGD;
SURVEY 8(f) f3).  The fused path uses the same dW accumulation and the same fp32 fma as
tgp_backward + tgp_step, so every parameter after the step is compared BITWISE with the unfused
path, over several steps (graph replay, a changed learning rate, dropout); and once against the
fp64 oracle (normwise 2e-2, reading Z15)."""
import numpy as np
import pytest

from synth import configs as C

from _gpu import make_case, oracle_step

pytestmark = pytest.mark.gpu


def _train(layers, params, x, t, *, m, n, ckpt, dtype, lrs, fused, seed=3, balance=None):
    import torch

    from paper_2004_09910_b200 import Pipeline

    B = x.shape[0]
    P = Pipeline(layers, chunks=m, devices=[0] * n, balance=balance, checkpoint=ckpt, max_batch=B, dtype=dtype,
                 seed=seed)
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


def _bitwise(layers, B, m, n, ckpt, dtype, lrs, balance=None):
    x, t, params = make_case(layers, B, 5, dtype)
    a = _train(layers, params, x, t, m=m, n=n, ckpt=ckpt, dtype=dtype, lrs=lrs, fused=False, balance=balance)
    b = _train(layers, params, x, t, m=m, n=n, ckpt=ckpt, dtype=dtype, lrs=lrs, fused=True, balance=balance)
    assert a["losses"] == b["losses"]
    assert np.array_equal(a["dx"], b["dx"])
    for k, (pa, pb) in enumerate(zip(a["params"], b["params"])):
        assert np.array_equal(pa, pb), k
    # the steps really changed the weights
    assert not np.array_equal(a["params"][2], params[2])


def test_fused_bitwise_stream_kernel_shapes():
    # 2 partitions of RESMLP blocks (stream kernel), dropout, three steps with two learning rates
    _bitwise(C.resmlp_stack(4, 512, hidden=1024, dropout=0.1), 64, 4, 2, "except_last", "bf16", [0.05, 0.05, 0.02])


def test_fused_bitwise_mixed_layers_and_ragged_batch():
    # U-MLP: MERGE / LINEAR layers take the unfused path inside the fused task; ragged micro-batches
    layers = C.umlp(d=256, levels=2, blocks_per_level=1, mid_blocks=1)
    _bitwise(layers, 40, 3, 2, "always", "bf16", [0.05, 0.03])


def test_fused_bitwise_full_c2_width():
    # the bench's block shape: d = H = 4096, B = 512, m = 32 (4 of the 32 blocks)
    _bitwise(C.resmlp_stack(4, 4096), 512, 32, 1, "except_last", "bf16", [0.05, 0.05])


def test_fused_fp32_mode_falls_back_bitwise():
    _bitwise(C.mlp_chain(4, 64), 16, 4, 2, "always", "fp32", [0.1, 0.1])


def test_fused_matches_oracle():
    layers = C.resmlp_stack(3, 1024, hidden=2048, dropout=0.1)
    x, t, params = make_case(layers, 64, 8, "bf16")
    g = _train(layers, params, x, t, m=4, n=1, ckpt="except_last", dtype="bf16", lrs=[0.05], fused=True, seed=8)
    ref = oracle_step(layers, params, x, t, lr=0.05, m=4, seed=8, step=0)
    errs = {"loss": abs(g["losses"][0] - ref["loss"]) / abs(ref["loss"])}
    scale = max(np.max(np.abs(r)) for r in ref["grads"])
    for k, (pn, pr, p0) in enumerate(zip(g["params"], ref["params"], params)):
        pn = np.asarray(pn, np.float64).ravel()
        d_gpu = pn - np.asarray(p0, np.float64).ravel()
        d_ref = np.asarray(pr, np.float64).ravel() - np.asarray(p0, np.float64).ravel()
        excess = np.maximum(np.abs(d_gpu - d_ref) - 2.0 ** -24 * np.abs(pn), 0.0)
        errs[f"dtheta{k}"] = float(np.max(excess) / max(np.max(np.abs(d_ref)), 1e-3 * scale * 0.05))
    bad = {k: v for k, v in errs.items() if not v <= 2e-2}
    assert not bad, bad


def test_backward_step_after_pending_backward_is_a_state_error():
    import torch

    from paper_2004_09910_b200 import Pipeline, tgp

    layers = C.resmlp_stack(2, 512)
    P = Pipeline(layers, chunks=4, devices=[0], checkpoint="except_last", max_batch=64, dtype="bf16")
    X = torch.randn(64, 512, device="cuda")
    Y = torch.empty_like(X)
    DY = torch.randn_like(X)
    P.forward(X, 64, Y)
    P.backward(DY)
    P.forward(X, 64, Y)
    with pytest.raises(tgp.TgpError) as ei:
        P.backward_step(DY, 0.05)
    assert "(-2)" in str(ei.value)
    P.close()
