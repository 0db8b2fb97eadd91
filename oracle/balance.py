"""Partition balancer (§3, "a partition whose pairwise resource discrepancy is
small"; reading Z8: min-max contiguous block sum, lexicographically smallest boundaries on ties)
-- TEST INFRASTRUCTURE ONLY."""
import itertools


def balance_dp(costs, n):
    """Min-max contiguous partition of `costs` into n non-empty blocks by dynamic programming
    over prefix sums (O6).  Returns block sizes.  Ties: lexicographically smallest boundary
    vector, i.e. the first block as short as possible, then the second, ..."""
    L = len(costs)
    if not (1 <= n <= L):
        raise ValueError("need 1 <= n <= len(costs)")
    pre = [0.0]
    for c in costs:
        pre.append(pre[-1] + float(c))
    INF = float("inf")
    # best[p][e]: min over partitions of layers [e, L) into p blocks of the max block sum
    best = [[INF] * (L + 1) for _ in range(n + 1)]
    best[0][L] = 0.0
    for p in range(1, n + 1):
        for e in range(L - p, -1, -1):
            v = INF
            for end in range(e + 1, L - p + 2):
                blk = pre[end] - pre[e]
                v = min(v, max(blk, best[p - 1][end]))
            best[p][e] = v
    opt = best[n][0]
    # reconstruct: greedily take the smallest first block that still achieves the optimum
    sizes, e = [], 0
    for p in range(n, 0, -1):
        for end in range(e + 1, L - p + 2):
            if max(pre[end] - pre[e], best[p - 1][end]) <= opt:
                sizes.append(end - e)
                e = end
                break
    return sizes


def balance_brute(costs, n):
    """Exhaustive enumeration of all C(L-1, n-1) contiguous splits; lexicographic tie-break."""
    L = len(costs)
    best, best_b = None, None
    for cuts in itertools.combinations(range(1, L), n - 1):
        b = (0,) + cuts + (L,)
        mx = max(sum(costs[b[q]:b[q + 1]]) for q in range(n))
        if best is None or mx < best:
            best, best_b = mx, b
    return [best_b[q + 1] - best_b[q] for q in range(n)]


def block_max(costs, sizes):
    out, e = [], 0
    for s in sizes:
        out.append(sum(costs[e:e + s]))
        e += s
    return max(out)


def profile_size(layers, rows):
    """SPEC profile_size (§4.2.2: "parameters consume 8 bytes each for itself and
    its gradients"): per layer, 8 x its parameter count + the activation output of a `rows`-row
    sample in fp32 (rows x d_out x 4 bytes)."""
    from synth.configs import param_shapes
    import numpy as np
    shapes = param_shapes(layers)
    out = []
    for li, L in enumerate(layers):
        n = sum(int(np.prod(sh)) for (l, _, sh) in shapes if l == li)
        out.append(8.0 * n + rows * L["d_out"] * 4.0)
    return out
