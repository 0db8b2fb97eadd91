"""Pipeline emulator -- TEST INFRASTRUCTURE ONLY.

Executes the O5 record list in emitted order on micro-batches (fp64) with per-partition
state, exactly as the paper describes the tasks:
  F_{i,j}   x_i^j <- f^j(x_i^{j-1})                                  (Eq. F_{i,j})
  B_{i,j}   dx_i^{j-1} <- d_x f^j(dx_i^j);  g_i^j <- d_theta f^j(dx_i^j)  (Eq. B_{i,j})
  g^j = sum_i g_i^j
  F'_{i,j}  recomputation of F_{i,j} right before B_{i,j}, omitted for i = m
            under except_last; a checkpointed F keeps only its stage input (P:105,
            "memory consumption is reduced by a factor of m") plus the RNG key (seed, step).
  copies    COPY_F / COPY_B move boundary tensors (Alg. 1); SKIP_F / SKIP_B move
            a skip tensor directly s -> d and its gradient d -> s (portals, Fig. 6).

Asserts (raises AssertionError):
  * causality: every consumed buffer was produced by an earlier record;
  * a checkpointed F keeps exactly the stage input; live stash under `always` = m inputs;
  * F' output equals the discarded F output BITWISE (referential transparency, P:122 fn);
  * each skip tensor is copied exactly once per direction per micro-batch (0 if s == d).
"""
import numpy as np

from . import model as M
from .schedule import (B as K_B, COPY_B, COPY_F, F as K_F, RECOMPUTE, SKIP_B, SKIP_F, W as K_W,
                       checkpointed, records, route_partitions, split_offsets)


def emulate(layers, params, x, t, *, balance, m, mode, seed=0, step=0):
    n = len(balance)
    Bsz = x.shape[0]
    off = M.micro_offsets(layers, Bsz, m)
    P = M.group_params(layers, params)
    starts = [0]
    for c in balance:
        starts.append(starts[-1] + c)
    part_layers = [list(range(starts[j], starts[j + 1])) for j in range(n)]
    rparts = route_partitions(layers, balance)
    route_of_stash = {L["stash"]: li for li, L in enumerate(layers) if L["stash"] >= 0}
    route_of_pop = {L["pop"]: li for li, L in enumerate(layers) if L["pop"] >= 0}
    recs = records(m, n, mode, rparts)

    X = np.asarray(x, np.float64)
    out = {}          # (i, j) -> stage output
    recv = {}         # (i, j) -> received stage input (checkpoint slot; "shared memory")
    saved = {}        # (i, j) -> ("ckpt", input) | ("full", caches)
    fwd_out = {}      # (i, j) -> output of F (for the bitwise F' check)
    skip_src = {}     # (r, i) -> skip tensor at its source partition
    skip_dst = {}     # (r, i) -> skip tensor received at destination partition
    gin = {}          # (i, j) -> received output-gradient of stage j
    dxo = {}          # (i, j) -> input-gradient produced by B_{i,j}
    dskip_src = {}    # (r, i) -> skip gradient received at the source partition
    dskip_dst = {}    # (r, i) -> skip gradient produced at the destination partition
    gsum = [[None] * len(layers) for _ in range(m + 1)]
    dy_full = None
    loss = None
    done_B = set()
    copies = {"skip_f": 0, "skip_b": 0}
    bn_inputs = {}    # layer -> {i: x rows} (from F only, never F')

    def run_fwd(i, j, inp, collect_bn):
        rows = off[i] - off[i - 1]
        row0 = off[i - 1]
        h = inp
        caches = []
        local_skip = {}
        for li in part_layers[j - 1]:
            L = layers[li]
            s = None
            if L["pop"] >= 0:
                r = L["pop"]
                s = local_skip[r] if r in local_skip else skip_dst[(r, i)]
            if collect_bn and L["kind"] == "batchnorm":
                bn_inputs.setdefault(li, {})[i] = h.copy()
            y, c = M.layer_fwd(L, P[li], h, s, site=li, seed=seed, step=step, row0=row0,
                               groups=[(0, rows)])
            caches.append(c)
            if L["stash"] >= 0:
                r = L["stash"]
                if rparts[r][1] == j:
                    local_skip[r] = y
                else:
                    skip_src[(r, i)] = y
            h = y
        return h, caches

    for rec in recs:
        ph, k, kind, i, j, src, dst, r = [int(v) for v in rec]
        if kind == COPY_F:
            assert (i, src) in out, f"COPY_F before F_{i},{src}"
            recv[(i, j)] = out[(i, src)].copy()
        elif kind == SKIP_F:
            assert (r, i) in skip_src, f"SKIP_F of route {r} before its stash"
            skip_dst[(r, i)] = skip_src[(r, i)].copy()
            copies["skip_f"] += 1
        elif kind == K_F:
            inp = X[off[i - 1]:off[i]] if j == 1 else recv[(i, j)]
            y, caches = run_fwd(i, j, inp, True)
            out[(i, j)] = y
            fwd_out[(i, j)] = y.copy()
            if checkpointed(i, m, mode):
                saved[(i, j)] = ("ckpt", inp)          # only the stage input is kept
            else:
                saved[(i, j)] = ("full", caches)
        elif kind == RECOMPUTE:
            if i < m:
                assert (i + 1, j) in done_B, f"F'_{i},{j} before B_{i+1},{j}"
            tag, inp = saved[(i, j)]
            assert tag == "ckpt"
            y, caches = run_fwd(i, j, inp, False)
            assert np.array_equal(y, fwd_out[(i, j)]), "F' != F (referential transparency)"
            saved[(i, j)] = ("full", caches)
        elif kind == COPY_B:
            assert (i, src) in dxo, f"COPY_B before B_{i},{src}"
            gin[(i, j)] = dxo[(i, src)].copy()
        elif kind == SKIP_B:
            assert (r, i) in dskip_dst, f"SKIP_B of route {r} before its pop's backward"
            dskip_src[(r, i)] = dskip_dst[(r, i)].copy()
            copies["skip_b"] += 1
        elif kind == K_B:
            if j == n and dy_full is None:
                assert all((ii, n) in out for ii in range(1, m + 1)), "loss before all outputs"
                y_all = np.concatenate([out[(ii, n)] for ii in range(1, m + 1)], axis=0)
                loss, dy_full = M.loss_fn(layers, y_all, t)
            if i < m:
                assert (i + 1, j) in done_B, "B order violated"
            tag, caches = saved[(i, j)]
            assert tag == "full", f"B_{i},{j} without activations"
            d = dy_full[off[i - 1]:off[i]] if j == n else gin[(i, j)]
            rows = off[i] - off[i - 1]
            local_dskip = {}
            for pos in range(len(part_layers[j - 1]) - 1, -1, -1):
                li = part_layers[j - 1][pos]
                L = layers[li]
                if L["stash"] >= 0:
                    rr = L["stash"]
                    d = d + (local_dskip.pop(rr) if rparts[rr][1] == j else dskip_src[(rr, i)])
                d, ds, g = M.layer_bwd(L, P[li], caches[pos], d, groups=[(0, rows)])
                if L["pop"] >= 0:
                    rr = L["pop"]
                    if rparts[rr][0] == j:
                        local_dskip[rr] = ds
                    else:
                        dskip_dst[(rr, i)] = ds
                gsum[i][li] = g
            dxo[(i, j)] = d
            done_B.add((i, j))
            del saved[(i, j)]
        elif kind == K_W:
            assert all((ii, j) in done_B for ii in range(1, m + 1)), "W before all B"
        # memory invariant under `always`: at most m saved stage inputs per partition
        if mode == "always":
            for jj in range(1, n + 1):
                assert sum(1 for (ii, pj), v in saved.items() if pj == jj and v[0] == "ckpt") <= m

    # g^j = sum_i g_i^j, ascending i
    grads = []
    for li in range(len(layers)):
        acc = None
        for i in range(1, m + 1):
            g = gsum[i][li]
            acc = [gg.copy() for gg in g] if acc is None else [a + gg for a, gg in zip(acc, g)]
        grads += acc
    n_cross = sum(1 for (s, d) in rparts if s != d)
    assert copies["skip_f"] == m * n_cross and copies["skip_b"] == m * n_cross
    y = np.concatenate([out[(ii, n)] for ii in range(1, m + 1)], axis=0)
    dx = np.concatenate([dxo[(ii, 1)] for ii in range(1, m + 1)], axis=0)
    bn = []
    for li, L in enumerate(layers):
        if L["kind"] == "batchnorm":
            xf = np.concatenate([bn_inputs[li][ii] for ii in range(1, m + 1)], axis=0)
            nb = xf.shape[0]
            mb = xf.mean(axis=0)
            vb = ((xf - mb) ** 2).mean(axis=0)
            bn.append((M.BN_MOMENTUM * mb, (1 - M.BN_MOMENTUM) + M.BN_MOMENTUM * vb * nb / (nb - 1)))
    return dict(loss=loss, y=y, grads=grads, dx=dx, bn=bn, copies=copies, records=recs)
