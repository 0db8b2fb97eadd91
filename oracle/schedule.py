"""Clock-cycle schedule of GPipe (§2.1-2.2, §3.2.1 Alg. 1) -- TEST INFRASTRUCTURE ONLY.

Record encoding: 8 int32 (phase, clock, kind, i, j, src, dst, route),
i, j 1-based, route -1 except for skip records.
"""
import numpy as np

PH_FWD, PH_BWD, PH_W = 0, 1, 2
F, RECOMPUTE, B, COPY_F, COPY_B, SKIP_F, SKIP_B, W = range(8)
KIND_NAMES = {F: "F", RECOMPUTE: "R", B: "B", COPY_F: "COPY_F", COPY_B: "COPY_B",
              SKIP_F: "SKIP_F", SKIP_B: "SKIP_B", W: "W"}
MODES = ("always", "except_last", "never")


def split_sizes(B, m):
    """Micro-batch sizes ("x consists of m smaller batches"; reading Z7 / SPEC S:323-327):
    ceil(B/m) for the first B mod m micro-batches, floor(B/m) for the rest."""
    if not (1 <= m <= B):
        raise ValueError("need 1 <= m <= B")
    q, r = divmod(B, m)
    return [q + 1 if i < r else q for i in range(m)]


def split_offsets(B, m):
    s = split_sizes(B, m)
    off = [0]
    for v in s:
        off.append(off[-1] + v)
    return off  # m+1 entries, micro-batch i (1-based) = rows [off[i-1], off[i])


def clock(k, m, n):
    """Tasks of forward clock k (Alg. 1): {(i,j) : i+j-1 = k}, ascending j (Z1)."""
    return [(k - j + 1, j) for j in range(max(1, k - m + 1), min(k, n) + 1)]


def checkpointed(i, m, mode):
    """Is micro-batch i checkpointed?  always: all; except_last: i < m (P:108, P:305 fn);
    never: none (Z4)."""
    if mode == "always":
        return True
    if mode == "except_last":
        return i < m
    if mode == "never":
        return False
    raise ValueError(mode)


def records(m, n, mode, routes=None):
    """The O5 record list.  `routes` = list of (s, d) partition pairs (1-based), route id = index.

    Forward clock k = 1..m+n-1 (Alg. 1): all copies of the clock first, then the
    computes.  Backward clock k' = 1..m+n-1 mirrors it: tasks {i+j-1 = m+n-k'} in descending j
    (Z2); copies first (Z5); each B_{i,j} preceded by F'_{i,j} if checkpointed (Z3).
    Skip copies ride in the clock of the consumer task (Z6).  Phase 2: deferred dW per partition.
    """
    routes = list(routes or [])
    out = []
    T = m + n - 1
    for k in range(1, T + 1):
        tasks = clock(k, m, n)
        for (i, j) in tasks:
            if j > 1:
                out.append((PH_FWD, k, COPY_F, i, j, j - 1, j, -1))
        for (i, d) in tasks:
            for r, (s, dd) in enumerate(routes):
                if dd == d and s != d:
                    out.append((PH_FWD, k, SKIP_F, i, d, s, d, r))
        for (i, j) in tasks:
            out.append((PH_FWD, k, F, i, j, j, j, -1))
    for kp in range(1, T + 1):
        tasks = list(reversed(clock(m + n - kp, m, n)))
        for (i, j) in tasks:
            if j < n:
                out.append((PH_BWD, kp, COPY_B, i, j, j + 1, j, -1))
        for (i, s) in tasks:
            for r, (ss, d) in enumerate(routes):
                if ss == s and s != d:
                    out.append((PH_BWD, kp, SKIP_B, i, s, d, s, r))
        for (i, j) in tasks:
            if checkpointed(i, m, mode):
                out.append((PH_BWD, kp, RECOMPUTE, i, j, j, j, -1))
            out.append((PH_BWD, kp, B, i, j, j, j, -1))
    for j in range(1, n + 1):
        out.append((PH_W, 0, W, 0, j, j, j, -1))
    return np.array(out, dtype=np.int32).reshape(-1, 8)


def device_order(recs, j):
    """Per-partition projection onto compute tasks (O11 / Fig. 3): list of (kind, i)."""
    return [(int(r[2]), int(r[3])) for r in recs if r[2] in (F, RECOMPUTE, B, W) and r[4] == j]


def route_partitions(layers, balance):
    """Map layer-index skip routes to (source partition, destination partition), 1-based."""
    part_of = []
    for j, c in enumerate(balance):
        part_of += [j + 1] * c
    st, po = {}, {}
    for li, L in enumerate(layers):
        if L["stash"] >= 0:
            st[L["stash"]] = li
        if L["pop"] >= 0:
            po[L["pop"]] = li
    return [(part_of[st[r]], part_of[po[r]]) for r in sorted(st)]
