"""Pins for oracle/model.py and oracle/emulator.py.

  * central finite differences (fp64) on tiny models -- independent of the VJP formulas;
  * torch.autograd fp64 on CPU (an independent library implementation of the same forward);
  * BatchNorm running statistics vs torch.nn.functional.batch_norm on the full mini-batch;
  * emulator (micro-batched, O5 order) == full batch within 1e-12 normwise (P:70 g = sum_i g_i),
    F' == F bitwise (checked inside the emulator).
"""
import itertools

import numpy as np
import pytest
import torch

from oracle import model as M
from oracle.emulator import emulate
from oracle.philox import dropout_keep
from synth import configs as C
from synth import gen as G


def nwise(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def tiny_resmlp(d=8):
    return [C.layer("resmlp", d, d, d_hidden=12, act="gelu"),
            C.layer("resmlp", d, d, d_hidden=6, act="gelu", dropout=0.25),
            C.layer("linear", d, 5, act="relu")]


def tiny_umlp(d=6):
    return C.umlp(d=d, levels=2, blocks_per_level=1, mid_blocks=1)


def tiny_ln(d=7):
    return C.ln_mlp(2, d, dropout=0.3)


def tiny_bn(d=5):
    return [C.layer("linear", d, d), C.layer("batchnorm", d, d, act="relu"),
            C.layer("linear", d, d), C.layer("batchnorm", d, d, act="none")]


def _loss(layers, params, x, t, m, seed, step):
    y, _ = M.forward(layers, params, x, m=m, seed=seed, step=step)
    return M.mse(y, t)[0]


@pytest.mark.parametrize("mk,m", [(tiny_resmlp, 1), (tiny_umlp, 1), (tiny_bn, 2), (tiny_ln, 2)])
def test_finite_differences(mk, m):
    layers = mk()
    x, t = G.inputs(layers, 4, seed=11)
    params = [p.astype(np.float64) for p in G.params(layers, seed=11)]
    x = x.astype(np.float64)
    r = M.train_step(layers, params, x, t, lr=0.0, m=m, seed=99, step=3)
    h = 1e-6
    rs = np.random.default_rng(0)
    for pi, p in enumerate(params):
        gfd = np.zeros_like(p)
        flat = p.reshape(-1)
        idxs = rs.choice(flat.size, size=min(flat.size, 12), replace=False)
        for q in idxs:
            old = flat[q]
            flat[q] = old + h
            lp = _loss(layers, params, x, t, m, 99, 3)
            flat[q] = old - h
            lm = _loss(layers, params, x, t, m, 99, 3)
            flat[q] = old
            gfd.reshape(-1)[q] = (lp - lm) / (2 * h)
        ga = r["grads"][pi].reshape(-1)[idxs]
        gf = gfd.reshape(-1)[idxs]
        assert np.max(np.abs(ga - gf)) <= 1e-6 * max(1.0, np.max(np.abs(gf))) + 1e-9, pi
    # input gradient too
    xf = x.copy()
    for q in range(3):
        e = np.zeros_like(xf)
        e.reshape(-1)[q * 5] = h
        d = (_loss(layers, params, xf + e, t, m, 99, 3) - _loss(layers, params, xf - e, t, m, 99, 3)) / (2 * h)
        assert abs(d - r["dx"].reshape(-1)[q * 5]) < 1e-7


# ---------------------------------------------------------------- torch fp64 cross-check
def torch_step(layers, params, x, t, m, seed, step, lr=None):
    P = [torch.tensor(np.asarray(p, np.float64), requires_grad=True) for p in params]
    X = torch.tensor(np.asarray(x, np.float64), requires_grad=True)
    B = X.shape[0]
    off = [0]
    q, rr = divmod(B, m)
    for i in range(m):
        off.append(off[-1] + q + (1 if i < rr else 0))
    act = {"none": lambda z: z, "relu": torch.relu,
           "gelu": lambda z: torch.nn.functional.gelu(z, approximate="none")}
    h = X
    k = 0
    skips = {}
    running = []
    for li, L in enumerate(layers):
        if L["kind"] in ("linear", "merge"):
            W, b = P[k], P[k + 1]
            k += 2
            xin = torch.cat([h, skips[L["pop"]]], dim=1) if L["kind"] == "merge" else h
            y = act[L["act"]](torch.nn.functional.linear(xin, W, b))
            if L["dropout"] > 0:
                keep = torch.tensor(dropout_keep(seed, step, li, 0, B, y.shape[1], L["dropout"]))
                y = y * keep / (1 - L["dropout"])
        elif L["kind"] == "resmlp":
            g_, b_, W1, b1, W2, b2 = P[k:k + 6]
            k += 6
            hh = torch.nn.functional.layer_norm(h, (h.shape[1],), g_, b_, eps=1e-5)
            g = act[L["act"]](torch.nn.functional.linear(hh, W1, b1))
            if L["dropout"] > 0:
                keep = torch.tensor(dropout_keep(seed, step, li, 0, B, g.shape[1], L["dropout"]))
                g = g * keep / (1 - L["dropout"])
            y = h + torch.nn.functional.linear(g, W2, b2)
        elif L["kind"] == "layernorm":
            g_, b_ = P[k:k + 2]
            k += 2
            y = torch.nn.functional.layer_norm(h, (h.shape[1],), g_, b_, eps=1e-5)
        elif L["kind"] == "dropout":
            keep = torch.tensor(dropout_keep(seed, step, li, 0, B, h.shape[1], L["dropout"]))
            y = h * keep / (1 - L["dropout"])
        elif L["kind"] == "batchnorm":
            g_, b_ = P[k:k + 2]
            k += 2
            parts = [torch.nn.functional.batch_norm(h[off[i]:off[i + 1]], None, None, g_, b_,
                                                    training=True, eps=1e-5) for i in range(m)]
            y = act[L["act"]](torch.cat(parts, 0))
            rm = torch.zeros(h.shape[1], dtype=torch.float64)
            rv = torch.ones(h.shape[1], dtype=torch.float64)
            torch.nn.functional.batch_norm(h.detach(), rm, rv, None, None, training=True,
                                           momentum=0.1, eps=1e-5)
            running.append((rm.numpy(), rv.numpy()))
        if L["stash"] >= 0:
            skips[L["stash"]] = y
        h = y
    T = torch.tensor(np.asarray(t, np.float64))
    loss = ((h - T) ** 2).sum() / T.numel()
    loss.backward()
    grads = [p.grad.numpy().copy() for p in P]
    if lr is None:
        return float(loss.detach()), grads, X.grad.numpy(), running
    # the optimizer step by an independent library routine: plain SGD, no momentum / decay
    opt = torch.optim.SGD(P, lr=lr, momentum=0.0, weight_decay=0.0)
    opt.step()
    return float(loss.detach()), grads, X.grad.numpy(), running, [p.detach().numpy() for p in P]


@pytest.mark.parametrize("name", ["C1", "C2small", "C2small_drop", "C4small", "BN", "LN"])
def test_vs_torch_autograd(name):
    if name == "C1":
        cfg = C.C1()
        layers, B, m = cfg.layers, cfg.batch, 1
    elif name == "C2small":
        layers, B, m = C.resmlp_stack(8, 256), 64, 1
    elif name == "C2small_drop":
        layers, B, m = C.resmlp_stack(4, 128, dropout=0.1), 32, 1
    elif name == "C4small":
        layers, B, m = C.umlp(d=64), 16, 1
    elif name == "LN":
        layers, B, m = C.ln_mlp(3, 64, dropout=0.2), 24, 3
    else:
        cfg = C.BN()
        layers, B, m = cfg.layers, cfg.batch, cfg.m
    x, t = G.inputs(layers, B, seed=5)
    params = G.params(layers, seed=5)
    r = M.train_step(layers, params, x, t, lr=0.1, m=m, seed=77, step=2)
    loss, grads, dx, running, new = torch_step(layers, params, x, t, m, 77, 2, lr=0.1)
    assert abs(r["loss"] - loss) <= 1e-12 * abs(loss)
    scale = max(np.max(np.abs(gt)) for gt in grads)  # BN makes the preceding bias grad exactly 0
    for g, gt in zip(r["grads"], grads):
        assert np.max(np.abs(g - gt)) <= 1e-11 * max(np.max(np.abs(gt)), 1e-3 * scale)
    assert nwise(r["dx"], dx) <= 1e-11
    for (rm, rv), (tm, tv) in zip(r["bn"], running):
        assert nwise(rm, tm) <= 1e-12 and nwise(rv, tv) <= 1e-12
    # the SGD update pinned against torch.optim.SGD (VERDICT r1 "weak" 3): theta' and delta-theta
    for p, pn, pt in zip(params, r["params"], new):
        p = np.asarray(p, np.float64)
        assert np.max(np.abs(pn - pt)) <= 1e-11 * max(np.max(np.abs(pt - p)), 1e-3 * scale * 0.1)


# ---------------------------------------------------------------- emulator (O10)
def _bal(L, n):
    q, r = divmod(L, n)
    return [q + (1 if j < r else 0) for j in range(n)]


@pytest.mark.parametrize("m,n,mode", list(itertools.product([1, 2, 4, 8], [1, 2, 4], ["always", "except_last", "never"])))
def test_emulator_equals_full_batch_mlp8(m, n, mode):
    # SPEC acceptance 1 grid on an 8-layer MLP (with dropout on two layers)
    layers = C.mlp_chain(8, 6, act="gelu")
    layers[2]["dropout"] = 0.3
    layers[5]["dropout"] = 0.2
    B = 16
    x, t = G.inputs(layers, B, seed=3)
    params = G.params(layers, seed=3)
    full = M.train_step(layers, params, x, t, lr=0.0, m=1, seed=9, step=4)
    em = emulate(layers, params, x, t, balance=_bal(8, n), m=m, mode=mode, seed=9, step=4)
    assert abs(em["loss"] - full["loss"]) <= 1e-12 * abs(full["loss"])
    for g, gf in zip(em["grads"], full["grads"]):
        assert nwise(g, gf) <= 1e-12
    assert nwise(em["dx"], full["dx"]) <= 1e-12


@pytest.mark.parametrize("m,n,mode", list(itertools.product([1, 2, 4], [1, 2, 4], ["always", "except_last", "never"])))
def test_emulator_equals_full_batch_umlp(m, n, mode):
    layers = tiny_umlp(8)
    layers[1]["dropout"] = 0.1
    x, t = G.inputs(layers, 8, seed=4)
    params = G.params(layers, seed=4)
    full = M.train_step(layers, params, x, t, lr=0.0, m=1, seed=1, step=0)
    em = emulate(layers, params, x, t, balance=_bal(len(layers), n), m=m, mode=mode, seed=1, step=0)
    for g, gf in zip(em["grads"], full["grads"]):
        assert nwise(g, gf) <= 1e-12
    assert nwise(em["dx"], full["dx"]) <= 1e-12


@pytest.mark.parametrize("m,n", [(1, 2), (2, 2), (4, 2), (4, 4)])
def test_emulator_bn_matches_microbatch_bn(m, n):
    # BN is intra-batch (P:56 footnote): the pipelined run equals the full-batch oracle only when
    # the oracle also uses per-micro-batch statistics (O9); running stats from the full batch.
    cfg = C.BN()
    layers = cfg.layers
    x, t = G.inputs(layers, 16, seed=8)
    params = G.params(layers, seed=8)
    full = M.train_step(layers, params, x, t, lr=0.0, m=m)
    em = emulate(layers, params, x, t, balance=_bal(len(layers), n), m=m, mode="except_last")
    scale = max(np.max(np.abs(gf)) for gf in full["grads"])
    for g, gf in zip(em["grads"], full["grads"]):
        assert np.max(np.abs(g - gf)) <= 1e-12 * max(np.max(np.abs(gf)), 1e-3 * scale)
    for (a, b), (c, d) in zip(em["bn"], full["bn"]):
        assert nwise(a, c) <= 1e-12 and nwise(b, d) <= 1e-12
    if m > 1:
        # and it is NOT the full-batch-statistics BN (the paper's "not identical anymore")
        ref1 = M.train_step(layers, params, x, t, lr=0.0, m=1)
        assert max(nwise(g, gf) for g, gf in zip(em["grads"], ref1["grads"])) > 1e-6


def test_emulator_detects_recompute_mismatch():
    # negative control for the bitwise F' check: a non-referentially-transparent layer is caught
    layers = C.mlp_chain(2, 4)
    x, t = G.inputs(layers, 4, seed=1)
    params = G.params(layers, seed=1)
    calls = {"n": 0}
    orig = M.layer_fwd

    def flaky(L, p, xx, s, **kw):
        calls["n"] += 1
        y, c = orig(L, p, xx, s, **kw)
        if calls["n"] > 4:   # every recompute differs
            y = y + 1e-9
        return y, c

    M.layer_fwd = flaky
    try:
        with pytest.raises(AssertionError):
            emulate(layers, params, x, t, balance=[1, 1], m=2, mode="always")
    finally:
        M.layer_fwd = orig
