"""Pins for the GPT-2-shaped oracle layers (C5; oracle/model.py embed / transformer / lmhead / CE).

  * attention forward == torch.nn.functional.scaled_dot_product_attention(is_causal=True) (fp64,
    an independent library routine), per head, dropout off;
  * the whole embed + blocks + LM head + CE step == torch.autograd fp64 on CPU (forward written
    with torch.nn.functional primitives; dropout masks from the Philox generator, itself pinned by
    known-answer vectors in test_oracle_balance_philox.py);
  * central finite differences on a tiny model, with dropout;
  * the micro-batched emulator (O5 order, F' bitwise) == full batch within 1e-12.
"""
import numpy as np
import pytest
import torch
import torch.nn.functional as F

from oracle import model as M
from oracle.emulator import emulate
from oracle.philox import dropout_keep
from synth import configs as C
from synth import gen as G


def nwise(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def tiny(dropout=0.0, d=8, nh=2, seq=4, V=7, blocks=2):
    return C.gpt2_stack(blocks, d, nh, seq, V, dropout)


def test_attention_matches_sdpa():
    rs = np.random.default_rng(3)
    nh, seq, dh = 3, 16, 8
    d = nh * dh
    qkv = rs.standard_normal((2 * seq, 3 * d))
    ctx, _ = M._attn_fwd(qkv, nh, seq, 0.0, 0, 0, 0, 0)
    for s in range(2):
        for h in range(nh):
            rows = slice(s * seq, (s + 1) * seq)
            q, k, v = (torch.tensor(qkv[rows, o + h * dh:o + (h + 1) * dh]) for o in (0, d, 2 * d))
            ref = F.scaled_dot_product_attention(q[None], k[None], v[None], is_causal=True)[0]
            assert np.max(np.abs(ctx[rows, h * dh:(h + 1) * dh] - ref.numpy())) < 1e-13


def test_cross_entropy_matches_torch():
    rs = np.random.default_rng(4)
    y = rs.standard_normal((10, 7)) * 3
    t = rs.integers(0, 7, 10)
    loss, dy = M.cross_entropy(y, t)
    yt = torch.tensor(y, requires_grad=True)
    lt = F.cross_entropy(yt, torch.tensor(t))
    lt.backward()
    assert abs(loss - lt.item()) < 1e-14
    assert np.max(np.abs(dy - yt.grad.numpy())) < 1e-15


def _torch_step(layers, params, x, t, seed, step):
    """The same model written with torch primitives; returns loss and grads (fp64, autograd)."""
    P = [torch.tensor(np.asarray(p, np.float64), requires_grad=True) for p in params]
    k = 0
    T = x.shape[0]
    h = None
    for li, L in enumerate(layers):
        p = L["dropout"]

        def drop(a, site):
            if p <= 0:
                return a
            keep = torch.tensor(dropout_keep(seed, step, site, 0, a.shape[0], a.shape[1], p))
            return a * keep / (1 - p)

        if L["kind"] == "embed":
            wte, wpe = P[k:k + 2]
            k += 2
            ids = torch.tensor(np.rint(x[:, 0]).astype(np.int64))
            pos = torch.arange(T) % L["seq"]
            h = drop(F.embedding(ids, wte) + F.embedding(pos, wpe), li)
        elif L["kind"] == "transformer":
            g1, b1n, Wqkv, bqkv, Wo, bo, g2, b2n, W1, b1, W2, b2 = P[k:k + 12]
            k += 12
            d, nh, seq = L["d_in"], L["n_heads"], L["seq"]
            dh = d // nh
            a = F.linear(F.layer_norm(h, (d,), g1, b1n, eps=1e-5), Wqkv, bqkv)
            q, kk, v = a[:, :d], a[:, d:2 * d], a[:, 2 * d:]
            ns = T // seq
            sh = lambda u: u.reshape(ns, seq, nh, dh).permute(0, 2, 1, 3)  # [ns, nh, seq, dh]
            S = sh(q) @ sh(kk).transpose(-1, -2) / np.sqrt(dh)
            S = S.masked_fill(~torch.tril(torch.ones(seq, seq, dtype=torch.bool)), float("-inf"))
            Pm = torch.softmax(S, dim=-1)
            if p > 0:
                keep = torch.tensor(dropout_keep(seed, step, li + M.SITE_ATTN, 0, ns * nh * seq, seq, p))
                Pm = Pm * keep.reshape(ns, nh, seq, seq) / (1 - p)
            ctx = (Pm @ sh(v)).permute(0, 2, 1, 3).reshape(T, d)
            x1 = h + drop(F.linear(ctx, Wo, bo), li + M.SITE_RES1)
            z = F.linear(F.layer_norm(x1, (d,), g2, b2n, eps=1e-5), W1, b1)
            h = x1 + drop(F.linear(F.gelu(z), W2, b2), li + M.SITE_RES2)
        elif L["kind"] == "lmhead":
            g, b, W = P[k:k + 3]
            k += 3
            h = F.linear(F.layer_norm(h, (L["d_in"],), g, b, eps=1e-5), W)
    loss = F.cross_entropy(h, torch.tensor(np.asarray(t, np.int64)))
    loss.backward()
    return loss.item(), [q.grad.numpy() for q in P]


@pytest.mark.parametrize("dropout", [0.0, 0.2])
def test_gpt2_step_matches_torch_autograd(dropout):
    layers = tiny(dropout, d=16, nh=2, seq=8, V=11, blocks=2)
    x, t = G.inputs(layers, 3, seed=5)
    params = [p.astype(np.float64) for p in G.params(layers, seed=5)]
    r = M.train_step(layers, params, x, t, lr=0.0, seed=9, step=2)
    lt, gt = _torch_step(layers, params, x, t, 9, 2)
    assert abs(r["loss"] - lt) < 1e-12
    for a, b in zip(r["grads"], gt):
        assert nwise(a, b) < 1e-11


def test_gpt2_finite_differences():
    layers = tiny(0.25)
    x, t = G.inputs(layers, 2, seed=7)
    params = [p.astype(np.float64) for p in G.params(layers, seed=7)]
    r = M.train_step(layers, params, x, t, lr=0.0, seed=3, step=1)

    def loss():
        y, _ = M.forward(layers, params, x, seed=3, step=1)
        return M.cross_entropy(y, t)[0]

    h = 1e-6
    rs = np.random.default_rng(0)
    for pi, p in enumerate(params):
        flat = p.reshape(-1)
        for q in rs.choice(flat.size, size=min(flat.size, 6), replace=False):
            old = flat[q]
            flat[q] = old + h
            lp = loss()
            flat[q] = old - h
            lm = loss()
            flat[q] = old
            fd = (lp - lm) / (2 * h)
            assert abs(r["grads"][pi].reshape(-1)[q] - fd) <= 1e-7 + 1e-6 * abs(fd), (pi, q)


@pytest.mark.parametrize("mode", ["always", "except_last", "never"])
@pytest.mark.parametrize("m,n", [(1, 1), (2, 2), (4, 3)])
def test_gpt2_pipelined_equals_full_batch(mode, m, n):
    layers = tiny(0.1, blocks=3)          # 5 layers
    x, t = G.inputs(layers, 4, seed=2)
    params = [p.astype(np.float64) for p in G.params(layers, seed=2)]
    bal = {1: [5], 2: [2, 3], 3: [2, 2, 1]}[n]
    full = M.train_step(layers, params, x, t, lr=0.0, m=m, seed=1, step=4)
    e = emulate(layers, params, x, t, balance=bal, m=m, mode=mode, seed=1, step=4)
    assert abs(e["loss"] - full["loss"]) < 1e-12
    for a, b in zip(e["grads"], full["grads"]):
        assert nwise(a, b) < 1e-12


def test_micro_offsets_whole_sequences():
    layers = tiny(seq=4)
    assert M.micro_offsets(layers, 5 * 4, 2) == [0, 12, 20]   # 5 samples -> [3, 2] (Z7)
    assert M.micro_offsets(C.mlp_chain(), 10, 4) == [0, 3, 6, 8, 10]
