"""BASELINE.json model configurations as plain data (SURVEY.md §8(d) "Concrete synthetic workloads").

A model is a list of layer dicts.  Keys:
  kind        "linear" | "resmlp" | "merge" | "batchnorm"
  d_in, d_out input / output feature width (for "merge": d_in is the width of the
              main input x; the popped skip tensor adds `d_skip` more input columns)
  d_hidden    hidden width of a "resmlp" block (W1: [d_hidden, d_in], W2: [d_out, d_hidden])
  act         "none" | "relu" | "gelu"   (applied after the affine map / normalisation)
  dropout     dropout probability applied after the activation (0.0 = none)
  stash       route id whose skip tensor is this layer's OUTPUT, or -1
  pop         route id consumed (concatenated after x) at this layer's INPUT, or -1
  d_skip      width of the popped skip tensor ("merge" only), else 0
  n_heads     attention heads ("transformer"), seq: tokens per sample ("embed", "transformer"),
  vocab       vocabulary size ("embed": d_in = 1, the token id; "lmhead": d_out = vocab)
  GPT-2-shaped kinds (C5): "embed", "transformer" (pre-LN block, MLP d_hidden, GELU,
  causal attention), "lmhead" (final LN + untied vocabulary projection, no bias)

A run is described by `Config` (layers + batch + m + n + checkpoint + dtype + lr).
Nothing here computes anything of the method; it is data only.
"""
from dataclasses import dataclass, field
from typing import List, Optional


def layer(kind, d_in, d_out, d_hidden=0, act="none", dropout=0.0, stash=-1, pop=-1, d_skip=0,
          n_heads=0, seq=0, vocab=0):
    return dict(kind=kind, d_in=int(d_in), d_out=int(d_out), d_hidden=int(d_hidden), act=act,
                dropout=float(dropout), stash=int(stash), pop=int(pop), d_skip=int(d_skip),
                n_heads=int(n_heads), seq=int(seq), vocab=int(vocab))


@dataclass
class Config:
    name: str
    layers: List[dict]
    batch: int
    m: int
    n: int
    checkpoint: str              # "always" | "except_last" | "never"
    dtype: str                   # "fp32" | "bf16"
    lr: float
    balance: Optional[List[int]] = None
    seed: int = 1234
    extra: dict = field(default_factory=dict)


def mlp_chain(n_layers=4, d=64, act="relu"):
    """C1 (BASELINE.json configs[0]): n_layers x [Linear(d->d, bias) + act]."""
    return [layer("linear", d, d, act=act) for _ in range(n_layers)]


def resmlp_stack(n_blocks=32, d=4096, hidden=None, dropout=0.0):
    """C2 (configs[1]): n_blocks x pre-LN residual MLP  y = x + W2 act(W1 LN(x) + b1) + b2."""
    hidden = d if hidden is None else hidden
    return [layer("resmlp", d, d, d_hidden=hidden, act="gelu", dropout=dropout) for _ in range(n_blocks)]


def umlp(d=2048, levels=4, blocks_per_level=2, mid_blocks=2, dropout=0.0):
    """C4 (configs[3]): U-Net-shaped MLP with long skip connections (stash/pop across stages).

    Encoder level l = 1..levels: `blocks_per_level` RESMLP blocks, the last one stashes route l-1.
    `mid_blocks` RESMLP blocks.  Decoder level l = levels..1: MERGE([x || pop s_l], 2d->d, GELU)
    followed by `blocks_per_level` RESMLP blocks.  Head Linear(d->d).
    """
    L = []
    for lvl in range(levels):
        for b in range(blocks_per_level):
            last = b == blocks_per_level - 1
            L.append(layer("resmlp", d, d, d_hidden=d, act="gelu", dropout=dropout,
                           stash=(lvl if last else -1)))
    for _ in range(mid_blocks):
        L.append(layer("resmlp", d, d, d_hidden=d, act="gelu", dropout=dropout))
    for lvl in reversed(range(levels)):
        L.append(layer("merge", d, d, act="gelu", pop=lvl, d_skip=d))
        for _ in range(blocks_per_level):
            L.append(layer("resmlp", d, d, d_hidden=d, act="gelu", dropout=dropout))
    L.append(layer("linear", d, d, act="none"))
    return L


def gpt2_stack(n_layers=48, d=1600, n_heads=25, seq=1024, vocab=50304, dropout=0.1):
    """C5 (configs[4]): embed + n_layers pre-LN GPT-2 blocks (MLP 4d, GELU) + final LN / LM head.
    The GPT-2 vocabulary (50257) is padded to 50304 = 393 x 128 (whole tensor-core tiles for the LM
    head; the padding rows are ordinary never-sampled tokens)."""
    L = [layer("embed", 1, d, dropout=dropout, seq=seq, vocab=vocab)]
    for _ in range(n_layers):
        L.append(layer("transformer", d, d, d_hidden=4 * d, act="gelu", dropout=dropout,
                       n_heads=n_heads, seq=seq))
    L.append(layer("lmhead", d, vocab, vocab=vocab))
    return L


def C5_small(n=2, m=4, checkpoint="always", dropout=0.1, batch=8):
    """Shrunk C5 (SURVEY 8(c) pins): 4 blocks, d = 128, 2 heads, seq 64, V = 512, B = 8 seqs."""
    return Config("C5s", gpt2_stack(4, 128, 2, 64, 512, dropout), batch=batch, m=m, n=n,
                  checkpoint=checkpoint, dtype="bf16", lr=0.01)


def C5(n=8, m=32, checkpoint="always", batch=32, n_layers=48):
    """Full C5: 48 x (d 1600, 25 heads, seq 1024), V 50304, 32 sequences, m = 32 (1 seq each)."""
    return Config("C5", gpt2_stack(n_layers), batch=batch, m=m, n=n, checkpoint=checkpoint, dtype="bf16",
                  lr=0.01)


def ln_mlp(n_blocks=2, d=256, dropout=0.1):
    """A sequence of plain layers with the standalone LayerNorm and Dropout kinds (any
    sequence of layers): n_blocks x [Linear(d->d, GELU), LayerNorm(d), Dropout(p)], Linear(d->d)."""
    out = []
    for _ in range(n_blocks):
        out += [layer("linear", d, d, act="gelu"), layer("layernorm", d, d), layer("dropout", d, d, dropout=dropout)]
    return out + [layer("linear", d, d)]


def bn_mlp(n=4, d=256):
    """BN micro-config: n x [Linear(d->d), BatchNorm(d), ReLU]."""
    L = []
    for _ in range(n):
        L.append(layer("linear", d, d, act="none"))
        L.append(layer("batchnorm", d, d, act="relu"))
    return L


def C1():
    return Config("C1", mlp_chain(4, 64), batch=16, m=4, n=2, checkpoint="always", dtype="fp32",
                  lr=0.1, balance=[2, 2])


def C2(n=8, m=32, checkpoint="except_last", blocks=32, d=4096, batch=512, dtype="bf16", dropout=0.0):
    return Config("C2", resmlp_stack(blocks, d, dropout=dropout), batch=batch, m=m, n=n,
                  checkpoint=checkpoint, dtype=dtype, lr=0.05, balance=[blocks // n] * n)


def C4(d=2048, batch=256, m=32, n=8, checkpoint="except_last", dtype="bf16"):
    return Config("C4", umlp(d), batch=batch, m=m, n=n, checkpoint=checkpoint, dtype=dtype, lr=0.05,
                  balance=[2, 3, 3, 3, 3, 3, 3, 3] if n == 8 else None)


def BN(m=4, n=2):
    return Config("BN", bn_mlp(4, 256), batch=64, m=m, n=n, checkpoint="except_last", dtype="fp32",
                  lr=0.05, balance=[4, 4] if n == 2 else None)


def param_shapes(layers):
    """Parameter tensors in canonical order (layer order; within a layer the order below).

    embed:     wte [vocab, d], wpe [seq, d]
    transformer: ln1 gamma, beta [d], Wqkv [3d, d], bqkv [3d], Wo [d, d], bo [d], ln2 gamma, beta [d],
               W1 [d_hidden, d], b1 [d_hidden], W2 [d, d_hidden], b2 [d]
    lmhead:    gamma [d], beta [d], W [vocab, d]
    linear:    W [d_out, d_in], b [d_out]
    merge:     W [d_out, d_in + d_skip], b [d_out]
    resmlp:    gamma [d_in], beta [d_in], W1 [d_hidden, d_in], b1 [d_hidden], W2 [d_out, d_hidden], b2 [d_out]
    batchnorm, layernorm: gamma [d], beta [d]
    dropout:   (no parameters)
    Returns a list of (layer_index, name, shape).
    """
    out = []
    for li, L in enumerate(layers):
        k = L["kind"]
        if k == "linear":
            out += [(li, "W", (L["d_out"], L["d_in"])), (li, "b", (L["d_out"],))]
        elif k == "merge":
            out += [(li, "W", (L["d_out"], L["d_in"] + L["d_skip"])), (li, "b", (L["d_out"],))]
        elif k == "resmlp":
            d, h = L["d_in"], L["d_hidden"]
            out += [(li, "gamma", (d,)), (li, "beta", (d,)), (li, "W1", (h, d)), (li, "b1", (h,)),
                    (li, "W2", (L["d_out"], h)), (li, "b2", (L["d_out"],))]
        elif k in ("batchnorm", "layernorm"):
            out += [(li, "gamma", (L["d_in"],)), (li, "beta", (L["d_in"],))]
        elif k == "dropout":
            pass
        elif k == "embed":
            out += [(li, "wte", (L["vocab"], L["d_out"])), (li, "wpe", (L["seq"], L["d_out"]))]
        elif k == "transformer":
            d, h = L["d_in"], L["d_hidden"]
            out += [(li, "gamma", (d,)), (li, "beta", (d,)), (li, "Wqkv", (3 * d, d)), (li, "bqkv", (3 * d,)),
                    (li, "Wo", (d, d)), (li, "bo", (d,)), (li, "gamma", (d,)), (li, "beta", (d,)),
                    (li, "W1", (h, d)), (li, "b1", (h,)), (li, "W2", (d, h)), (li, "b2", (d,))]
        elif k == "lmhead":
            out += [(li, "gamma", (L["d_in"],)), (li, "beta", (L["d_in"],)), (li, "W", (L["d_out"], L["d_in"]))]
        else:
            raise ValueError(k)
    return out


def routes(layers):
    """Skip routes as {route_id: (stash_layer, pop_layer)} (data lookup only)."""
    st, po = {}, {}
    for li, L in enumerate(layers):
        if L["stash"] >= 0:
            st[L["stash"]] = li
        if L["pop"] >= 0:
            po[L["pop"]] = li
    return {r: (st[r], po[r]) for r in sorted(st)}
