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
    return {"linear": 2, "merge": 2, "resmlp": 6, "batchnorm": 2}[L["kind"]]


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
    off = split_offsets(h.shape[0], m)
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
    loss, dy = mse(y, t)
    dx, grads = backward(layers, params, caches, dy)
    new = [np.asarray(p, np.float64) - lr * g for p, g in zip(params, grads)]
    return dict(loss=loss, y=y, dy=dy, grads=grads, params=new, dx=dx if want_dx else None,
                bn=bn_running(layers, caches))
