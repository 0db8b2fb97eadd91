"""Seeded input and parameter generators.  No method arithmetic here.

  rng(seed, tensor_id) = np.random.default_rng([seed, tensor_id])
  x, t           ~ N(0, 1)
  W, b           ~ U(-1/sqrt(fan_in), +1/sqrt(fan_in))
  gamma (LN/BN)  ~ 1 + 0.1 N(0, 1);  beta ~ 0.1 N(0, 1)

In bf16 mode every initial parameter and x are rounded to bf16-representable values
before either side sees them, so input rounding is not counted as error (O1).

Off-centre recipe (VERDICT r1 "What's weak" 2; stresses rounding points that depend on the
row mean, e.g. the LayerNorm folds R3/R4 of DESIGN.md):
  inputs(..., x_mean=mu)      x ~ N(mu, 1)
  params(..., ln="wide")      gamma ~ U(0.25, 4), beta ~ N(0, 1)
"""
import numpy as np

from .configs import param_shapes

# stable tensor-id enumeration
TID_X, TID_T = 1, 2
TID_PARAM0 = 1000


def rng(seed, tid):
    return np.random.default_rng([int(seed), int(tid)])


def round_bf16(a):
    """Round float array to the nearest bf16-representable value (RNE), returned as float32."""
    f = np.ascontiguousarray(a, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return (r & 0xFFFFFFFF).astype(np.uint32).view(np.float32)


def inputs(layers, batch, seed=1234, dtype="fp32", x_mean=0.0):
    """Return (x, t) float32 arrays [batch, d_in] and [batch, d_out].  GPT-2-shaped models (first
    layer "embed"): batch = sequences; x = token ids U{0..V-1} as float32 [batch*seq, 1],
    t = next-token targets int32 [batch*seq] (also U{0..V-1}; synthetic, no data)."""
    if layers[0]["kind"] == "embed":
        V, seq = layers[0]["vocab"], layers[0]["seq"]
        x = rng(seed, TID_X).integers(0, V, size=(batch * seq, 1)).astype(np.float32)
        t = rng(seed, TID_T).integers(0, V, size=(batch * seq,)).astype(np.int32)
        return x, t
    d_in, d_out = layers[0]["d_in"], layers[-1]["d_out"]
    x = (float(x_mean) + rng(seed, TID_X).standard_normal((batch, d_in))).astype(np.float32)
    t = rng(seed, TID_T).standard_normal((batch, d_out)).astype(np.float32)
    if dtype == "bf16":
        x = round_bf16(x)
    return x, t


def params(layers, seed=1234, dtype="fp32", ln="default", only=None):
    """Return the list of float32 parameter arrays in canonical order (configs.param_shapes).
    ln = "default" (gamma ~ 1 + 0.1 N, beta ~ 0.1 N) or "wide" (gamma ~ U(0.25, 4), beta ~ N(0, 1)).
    only: optional set of parameter indices to generate (None in the other slots; every tensor has
    its own seeded stream, so a subset is identical to the same entries of the full list)."""
    out = []
    for pid, (li, name, shape) in enumerate(param_shapes(layers)):
        if only is not None and pid not in only:
            out.append(None)
            continue
        g = rng(seed, TID_PARAM0 + pid)
        if name in ("wte", "wpe"):
            a = g.standard_normal(shape)
        elif name in ("W", "W1", "W2", "b", "b1", "b2", "Wqkv", "bqkv", "Wo", "bo"):
            if name in ("b", "b1", "b2", "bqkv", "bo"):
                fan_in = _fan_in(layers[li], name)
            else:
                fan_in = shape[1]
            bound = 1.0 / np.sqrt(fan_in)
            a = g.uniform(-bound, bound, size=shape)
        elif name == "gamma":
            a = g.uniform(0.25, 4.0, size=shape) if ln == "wide" else 1.0 + 0.1 * g.standard_normal(shape)
        elif name == "beta":
            a = g.standard_normal(shape) if ln == "wide" else 0.1 * g.standard_normal(shape)
        else:
            raise ValueError(name)
        a = a.astype(np.float32)
        if dtype == "bf16":
            a = round_bf16(a)
        out.append(a)
    return out


def _fan_in(L, name):
    if L["kind"] == "transformer":
        return L["d_hidden"] if name == "b2" else L["d_in"]
    if L["kind"] == "resmlp":
        return L["d_in"] if name == "b1" else L["d_hidden"]
    if L["kind"] == "merge":
        return L["d_in"] + L["d_skip"]
    return L["d_in"]
