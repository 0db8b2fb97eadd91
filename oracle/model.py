"""Full-batch fp64 training step of the layer sequence
-- TEST INFRASTRUCTURE ONLY.

GPipe is an execution-order transformation: "assuming that f does not involve any intra-batch
computation", the micro-batched forward F_{i,j} and backward B_{i,j} with
g^j = sum_i g_i^j reach exactly the full-batch result.  So the numeric oracle is the
plain definition: one unpipelined fp64 step on the whole mini-batch.  The two intra-batch
exceptions are handled as the paper/readings say:
  * BatchNorm (P:56 footnote, reading Z18): statistics per micro-batch in forward/backward;
    running statistics committed once from the full mini-batch (unbiased variance).
  * Dropout (reading Z17, O8): Philox masks keyed by the GLOBAL element index.

Layer formulas (O2) and textbook VJPs (O4):
  linear  z = x W^T + b, y = act(z) [* keep/(1-p)]
          dz = dy [* keep/(1-p)] * act'(z); dW = dz^T x; db = sum_rows dz; dx = dz W
  merge   as linear on [x || s] with W = [W_x | W_s]; dx = dz W_x, ds = dz W_s
  resmlp  mu, var (biased), r = (var + 1e-5)^-1/2, n = (x-mu) r, h = gamma n + beta,
          a = h W1^T + b1, g = act(a) [* keep/(1-p)], y = x + g W2^T + b2
  LN bwd  dgamma = sum dh*n, dbeta = sum dh, dn = dh*gamma,
          dx = r (dn - mean_row(dn) - n mean_row(dn*n))
  GELU    exact 0.5 a (1 + erf(a/sqrt 2));  GELU' = Phi(a) + a phi(a)
  ReLU'   [z > 0]  (derivative at 0 taken as 0)
  loss    L = sum (y-t)^2 / (B d_out);  dy = 2 (y-t) / (B d_out)   (O3, reading Z10)
  SGD     theta' = theta - lr g   ("trained by plain SGD")

GPT-2-shaped layers (C5, BASELINE.json configs[4]; reading Z13 -- the paper names GPT-2 1.5B as
a GPipe workload, but gives no formulas, so these are the textbook definitions).  Rows are
TOKENS; a sample is a sequence of `seq` tokens and micro-batches hold whole sequences.
  embed   y = wte[id] + wpe[pos] [* keep/(1-p)]   (id = token id carried in x[:, 0], pos = row % seq)
  block   h1 = LN1(x); qkv = h1 Wqkv^T + bqkv; per sequence and head (dh = d / n_heads):
          S = q k^T / sqrt(dh), causal (key <= query), P = softmax_row(S), Pd = P * keep/(1-p),
          ctx = Pd v; x1 = x + drop(ctx Wo^T + bo); h2 = LN2(x1); z = h2 W1^T + b1;
          y = x1 + drop(GELU(z) W2^T + b2)
          VJP of softmax: dS = P * (dP - rowsum(P * dP)), dP = dPd * keep/(1-p)
  lmhead  y = LN(x) W^T   (logits, no bias)
  CE      L = mean_t (logsumexp(y_t) - y_t[target_t]);  dy = (softmax(y) - onehot(target)) / T
Dropout sites (Philox counter word 2): embed / resmlp / linear: layer index; block: layer index
+ 1<<16 (attention probabilities, indexed in the [n_seq, n_heads, seq, seq] tensor), + 2<<16
(attention residual branch), + 3<<16 (MLP residual branch).
"""
import numpy as np
from scipy.special import erf

from .philox import dropout_keep
from .schedule import split_offsets

LN_EPS = 1e-5
BN_EPS = 1e-5
BN_MOMENTUM = 0.1
SQRT2 = np.sqrt(2.0)


def act_f(name, z):
    if name == "none":
        return z
    if name == "relu":
        return np.maximum(z, 0.0)
    if name == "gelu":
        return 0.5 * z * (1.0 + erf(z / SQRT2))
    raise ValueError(name)


def act_df(name, z):
    if name == "none":
        return np.ones_like(z)
    if name == "relu":
        return (z > 0).astype(np.float64)
    if name == "gelu":
        return 0.5 * (1.0 + erf(z / SQRT2)) + z * np.exp(-0.5 * z * z) / np.sqrt(2.0 * np.pi)
    raise ValueError(name)


def n_params(L):
    return {"linear": 2, "merge": 2, "resmlp": 6, "batchnorm": 2, "embed": 2, "transformer": 12,
            "lmhead": 3, "layernorm": 2, "dropout": 0}[L["kind"]]


def row_unit(layers):
    """Rows per sample: `seq` tokens for the GPT-2-shaped layers, else 1."""
    return max([int(L.get("seq", 0)) for L in layers] + [1])


def micro_offsets(layers, rows, m):
    """Row offsets of the m micro-batches: split the samples (reading Z7), then scale to rows."""
    u = row_unit(layers)
    assert rows % u == 0, "rows must be whole samples"
    return [o * u for o in split_offsets(rows // u, m)]


SITE_ATTN, SITE_RES1, SITE_RES2 = 1 << 16, 2 << 16, 3 << 16


def _ln_fwd(x, gamma, beta):
    mu = x.mean(axis=1, keepdims=True)
    var = ((x - mu) ** 2).mean(axis=1, keepdims=True)
    r = 1.0 / np.sqrt(var + LN_EPS)
    nrm = (x - mu) * r
    return gamma * nrm + beta, (r, nrm)


def _ln_bwd(dh, gamma, c):
    r, nrm = c
    dn = dh * gamma
    dx = r * (dn - dn.mean(axis=1, keepdims=True) - nrm * (dn * nrm).mean(axis=1, keepdims=True))
    return dx, (dh * nrm).sum(axis=0), dh.sum(axis=0)


def _attn_fwd(qkv, nh, seq, pdrop, seed, step, site, row0):
    """Causal multi-head attention on whole sequences; row0 = global token row of qkv[0]."""
    T, d3 = qkv.shape
    d = d3 // 3
    dh = d // nh
    ctx = np.zeros((T, d))
    cache = {}
    for s in range(T // seq):
        sg = (row0 // seq) + s                       # global sequence index
        rs = slice(s * seq, (s + 1) * seq)
        for h in range(nh):
            q = qkv[rs, h * dh:(h + 1) * dh]
            k = qkv[rs, d + h * dh:d + (h + 1) * dh]
            v = qkv[rs, 2 * d + h * dh:2 * d + (h + 1) * dh]
            S = q @ k.T / np.sqrt(dh)
            S = np.where(np.tril(np.ones((seq, seq), bool)), S, -np.inf)
            P = np.exp(S - S.max(axis=1, keepdims=True))
            P = P / P.sum(axis=1, keepdims=True)
            keep = None
            Pd = P
            if pdrop > 0:
                keep = dropout_keep(seed, step, site, (sg * nh + h) * seq, seq, seq, pdrop)
                Pd = P * keep / (1.0 - pdrop)
            ctx[rs, h * dh:(h + 1) * dh] = Pd @ v
            cache[(s, h)] = (P, keep)
    return ctx, cache


def _attn_bwd(qkv, dctx, nh, seq, pdrop, cache):
    T, d3 = qkv.shape
    d = d3 // 3
    dh = d // nh
    dqkv = np.zeros_like(qkv)
    for s in range(T // seq):
        rs = slice(s * seq, (s + 1) * seq)
        for h in range(nh):
            cq, ck, cv = (slice(o + h * dh, o + (h + 1) * dh) for o in (0, d, 2 * d))
            q, k, v = qkv[rs, cq], qkv[rs, ck], qkv[rs, cv]
            P, keep = cache[(s, h)]
            Pd = P if keep is None else P * keep / (1.0 - pdrop)
            do = dctx[rs, h * dh:(h + 1) * dh]
            dPd = do @ v.T
            dqkv[rs, cv] = Pd.T @ do
            dP = dPd if keep is None else dPd * keep / (1.0 - pdrop)
            dS = P * (dP - (P * dP).sum(axis=1, keepdims=True))
            dqkv[rs, cq] = dS @ k / np.sqrt(dh)
            dqkv[rs, ck] = dS.T @ q / np.sqrt(dh)
    return dqkv


def _drop(a, pdrop, seed, step, site, row0):
    if pdrop <= 0:
        return a, None
    keep = dropout_keep(seed, step, site, row0, a.shape[0], a.shape[1], pdrop)
    return a * keep / (1.0 - pdrop), keep


def _undrop(da, keep, pdrop):
    return da if keep is None else da * keep / (1.0 - pdrop)


def group_params(layers, params):
    out, k = [], 0
    for L in layers:
        c = n_params(L)
        out.append([np.asarray(p, dtype=np.float64) for p in params[k:k + c]])
        k += c
    assert k == len(params)
    return out


# ---------------------------------------------------------------- per-layer forward / backward
def layer_fwd(L, p, x, s, *, site, seed, step, row0, groups):
    """One layer on rows of the mini-batch.  x: [rows, d_in] fp64; s: popped skip or None;
    row0: global index of x's first row (dropout counters); groups: BN row groups (micro-batches)
    relative to x.  Returns (y, cache)."""
    k = L["kind"]
    pdrop = L["dropout"]
    rows = x.shape[0]
    if k in ("linear", "merge"):
        W, b = p
        xin = np.concatenate([x, s], axis=1) if k == "merge" else x
        z = xin @ W.T + b
        y = act_f(L["act"], z)
        keep = None
        if pdrop > 0:
            keep = dropout_keep(seed, step, site, row0, rows, y.shape[1], pdrop)
            y = y * keep / (1.0 - pdrop)
        return y, (xin, z, keep)
    if k == "resmlp":
        gamma, beta, W1, b1, W2, b2 = p
        mu = x.mean(axis=1, keepdims=True)
        var = ((x - mu) ** 2).mean(axis=1, keepdims=True)
        r = 1.0 / np.sqrt(var + LN_EPS)
        nrm = (x - mu) * r
        h = gamma * nrm + beta
        a = h @ W1.T + b1
        g = act_f(L["act"], a)
        keep = None
        if pdrop > 0:
            keep = dropout_keep(seed, step, site, row0, rows, g.shape[1], pdrop)
            g = g * keep / (1.0 - pdrop)
        y = x + g @ W2.T + b2
        return y, (x, r, nrm, h, a, g, keep)
    if k == "embed":
        wte, wpe = p
        ids = np.rint(x[:, 0]).astype(np.int64)
        pos = (row0 + np.arange(rows)) % L["seq"]
        y, keep = _drop(wte[ids] + wpe[pos], pdrop, seed, step, site, row0)
        return y, (ids, pos, keep)
    if k == "transformer":
        g1, be1, Wqkv, bqkv, Wo, bo, g2, be2, W1, b1, W2, b2 = p
        h1, c1 = _ln_fwd(x, g1, be1)
        qkv = h1 @ Wqkv.T + bqkv
        ctx, ca = _attn_fwd(qkv, L["n_heads"], L["seq"], pdrop, seed, step, site + SITE_ATTN, row0)
        ao, k1 = _drop(ctx @ Wo.T + bo, pdrop, seed, step, site + SITE_RES1, row0)
        x1 = x + ao
        h2, c2 = _ln_fwd(x1, g2, be2)
        z = h2 @ W1.T + b1
        g = act_f("gelu", z)
        mo, k2 = _drop(g @ W2.T + b2, pdrop, seed, step, site + SITE_RES2, row0)
        return x1 + mo, (h1, c1, qkv, ctx, ca, k1, x1, h2, c2, z, g, k2)
    if k == "lmhead":
        gamma, beta, W = p
        h, c = _ln_fwd(x, gamma, beta)
        return h @ W.T, (h, c)
    if k == "layernorm":  # standalone LayerNorm over the features of each row ("a sequence of layers")
        gamma, beta = p
        h, c = _ln_fwd(x, gamma, beta)
        return h, c
    if k == "dropout":  # standalone dropout: Philox mask of this layer's site (reading Z17)
        y, keep = _drop(x, pdrop, seed, step, site, row0)
        return y, keep
    if k == "batchnorm":
        gamma, beta = p
        y = np.empty_like(x)
        cache = []
        for (a0, a1) in groups:
            xb = x[a0:a1]
            mu = xb.mean(axis=0, keepdims=True)
            var = ((xb - mu) ** 2).mean(axis=0, keepdims=True)
            r = 1.0 / np.sqrt(var + BN_EPS)
            nrm = (xb - mu) * r
            z = gamma * nrm + beta
            y[a0:a1] = act_f(L["act"], z)
            cache.append((a0, a1, xb, r, nrm, z))
        return y, cache
    raise ValueError(k)


def layer_bwd(L, p, cache, dy, *, groups):
    """VJP of one layer.  Returns (dx, ds_or_None, [param grads])."""
    k = L["kind"]
    pdrop = L["dropout"]
    if k in ("linear", "merge"):
        W, b = p
        xin, z, keep = cache
        if keep is not None:
            dy = dy * keep / (1.0 - pdrop)
        dz = dy * act_df(L["act"], z)
        dW = dz.T @ xin
        db = dz.sum(axis=0)
        dxin = dz @ W
        if k == "merge":
            d = L["d_in"]
            return dxin[:, :d], dxin[:, d:], [dW, db]
        return dxin, None, [dW, db]
    if k == "resmlp":
        gamma, beta, W1, b1, W2, b2 = p
        x, r, nrm, h, a, g, keep = cache
        dW2 = dy.T @ g
        db2 = dy.sum(axis=0)
        dg = dy @ W2
        if keep is not None:
            dg = dg * keep / (1.0 - pdrop)
        da = dg * act_df(L["act"], a)
        dW1 = da.T @ h
        db1 = da.sum(axis=0)
        dh = da @ W1
        dgamma = (dh * nrm).sum(axis=0)
        dbeta = dh.sum(axis=0)
        dn = dh * gamma
        dx_ln = r * (dn - dn.mean(axis=1, keepdims=True) - nrm * (dn * nrm).mean(axis=1, keepdims=True))
        return dy + dx_ln, None, [dgamma, dbeta, dW1, db1, dW2, db2]
    if k == "embed":
        wte, wpe = p
        ids, pos, keep = cache
        de = _undrop(dy, keep, pdrop)
        dwte = np.zeros_like(wte)
        np.add.at(dwte, ids, de)
        dwpe = np.zeros_like(wpe)
        np.add.at(dwpe, pos, de)
        return np.zeros((dy.shape[0], 1)), None, [dwte, dwpe]
    if k == "transformer":
        g1, be1, Wqkv, bqkv, Wo, bo, g2, be2, W1, b1, W2, b2 = p
        h1, c1, qkv, ctx, ca, k1, x1, h2, c2, z, g, k2 = cache
        dm = _undrop(dy, k2, pdrop)                       # MLP branch
        dW2, db2 = dm.T @ g, dm.sum(axis=0)
        dz = (dm @ W2) * act_df("gelu", z)
        dW1, db1 = dz.T @ h2, dz.sum(axis=0)
        dx1_ln, dg2, dbe2 = _ln_bwd(dz @ W1, g2, c2)
        dx1 = dy + dx1_ln
        da = _undrop(dx1, k1, pdrop)                      # attention branch
        dWo, dbo = da.T @ ctx, da.sum(axis=0)
        dqkv = _attn_bwd(qkv, da @ Wo, L["n_heads"], L["seq"], pdrop, ca)
        dWqkv, dbqkv = dqkv.T @ h1, dqkv.sum(axis=0)
        dx_ln, dg1, dbe1 = _ln_bwd(dqkv @ Wqkv, g1, c1)
        return dx1 + dx_ln, None, [dg1, dbe1, dWqkv, dbqkv, dWo, dbo, dg2, dbe2, dW1, db1, dW2, db2]
    if k == "lmhead":
        gamma, beta, W = p
        h, c = cache
        dx, dg, db = _ln_bwd(dy @ W, gamma, c)
        return dx, None, [dg, db, dy.T @ h]
    if k == "layernorm":
        gamma, beta = p
        dx, dg, db = _ln_bwd(dy, gamma, cache)
        return dx, None, [dg, db]
    if k == "dropout":
        return _undrop(dy, cache, pdrop), None, []
    if k == "batchnorm":
        gamma, beta = p
        dx = np.empty_like(dy)
        dgamma = np.zeros_like(gamma)
        dbeta = np.zeros_like(beta)
        for (a0, a1, xb, r, nrm, z) in cache:
            dz = dy[a0:a1] * act_df(L["act"], z)
            dgamma += (dz * nrm).sum(axis=0)
            dbeta += dz.sum(axis=0)
            dn = dz * gamma
            dx[a0:a1] = r * (dn - dn.mean(axis=0, keepdims=True) - nrm * (dn * nrm).mean(axis=0, keepdims=True))
        return dx, None, [dgamma, dbeta]
    raise ValueError(k)


# ---------------------------------------------------------------- whole model
def forward(layers, params, x, *, m=1, seed=0, step=0, row0=0):
    """Forward over the full mini-batch (rows row0.. of the global batch).  Returns (y, caches)."""
    P = group_params(layers, params)
    h = np.asarray(x, dtype=np.float64)
    off = micro_offsets(layers, h.shape[0], m)
    groups = [(off[i], off[i + 1]) for i in range(m)]
    skips, caches = {}, []
    for li, L in enumerate(layers):
        s = skips[L["pop"]] if L["pop"] >= 0 else None
        y, c = layer_fwd(L, P[li], h, s, site=li, seed=seed, step=step, row0=row0, groups=groups)
        caches.append(c)
        if L["stash"] >= 0:
            skips[L["stash"]] = y
        h = y
    return h, (caches, groups)


def backward(layers, params, caches, dy):
    """Reverse pass.  Returns (dx, grads list in canonical order)."""
    P = group_params(layers, params)
    caches, groups = caches
    g_by_layer = [None] * len(layers)
    dskip = {}
    d = np.asarray(dy, dtype=np.float64)
    for li in range(len(layers) - 1, -1, -1):
        L = layers[li]
        if L["stash"] >= 0:
            d = d + dskip.pop(L["stash"])
        d, ds, g = layer_bwd(L, P[li], caches[li], d, groups=groups)
        if L["pop"] >= 0:
            dskip[L["pop"]] = ds
        g_by_layer[li] = g
    return d, [gg for g in g_by_layer for gg in g]


def mse(y, t):
    B, d = y.shape
    diff = y - np.asarray(t, dtype=np.float64)
    return float((diff ** 2).sum() / (B * d)), 2.0 * diff / (B * d)


def cross_entropy(y, t):
    """Mean token cross-entropy on logits y [T, V] with integer targets t [T] (O3, C5)."""
    T = y.shape[0]
    t = np.asarray(t).reshape(-1).astype(np.int64)
    mx = y.max(axis=1, keepdims=True)
    e = np.exp(y - mx)
    se = e.sum(axis=1, keepdims=True)
    lse = (mx + np.log(se))[:, 0]
    loss = float((lse - y[np.arange(T), t]).sum() / T)
    dy = e / se
    dy[np.arange(T), t] -= 1.0
    return loss, dy / T


def loss_fn(layers, y, t):
    """CE for models ending in an LM head, else MSE."""
    return cross_entropy(y, t) if layers[-1]["kind"] == "lmhead" else mse(y, t)


def bn_running(layers, caches, running=None):
    """Commit BN running statistics once per step from the full mini-batch (O9 / reading Z18):
    rm <- (1-mom) rm + mom mean_B;  rv <- (1-mom) rv + mom var_B * B/(B-1),
    mean_B, var_B the plain (biased) statistics of the whole mini-batch input of the layer."""
    caches, groups = caches
    out = []
    k = 0
    for li, L in enumerate(layers):
        if L["kind"] != "batchnorm":
            continue
        rm, rv = (np.zeros(L["d_in"]), np.ones(L["d_in"])) if running is None else running[k]
        k += 1
        xfull = np.concatenate([c[2] for c in caches[li]], axis=0)
        nb = xfull.shape[0]
        mean_B = xfull.mean(axis=0)
        var_B = ((xfull - mean_B) ** 2).mean(axis=0)
        out.append(((1 - BN_MOMENTUM) * rm + BN_MOMENTUM * mean_B,
                    (1 - BN_MOMENTUM) * rv + BN_MOMENTUM * var_B * nb / (nb - 1)))
    return out


def train_step(layers, params, x, t, *, lr, m=1, seed=0, step=0, want_dx=True):
    """One unpipelined fp64 training step on the whole mini-batch."""
    y, caches = forward(layers, params, x, m=m, seed=seed, step=step)
    loss, dy = loss_fn(layers, y, t)
    dx, grads = backward(layers, params, caches, dy)
    new = [np.asarray(p, np.float64) - lr * g for p, g in zip(params, grads)]
    return dict(loss=loss, y=y, dy=dy, grads=grads, params=new, dx=dx if want_dx else None,
                bn=bn_running(layers, caches))
