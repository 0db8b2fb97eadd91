"""Pins for oracle/schedule.py against what the paper fixes (Alg. 1) and closed forms."""
import itertools
import os

import numpy as np
import pytest

from oracle import schedule as S

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _parse_golden(name):
    out = {}
    for line in open(os.path.join(GOLD, name)):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        k, v = line.split(":", 1)
        out[int(k)] = v.split()
    return out


def test_clock_golden_m4_n3():
    g = _parse_golden("clock_cycles_m4_n3.txt")
    assert len(g) == 6
    for k, toks in g.items():
        want = [tuple(int(a) for a in t.strip("()").split(",")) for t in toks]
        assert S.clock(k, 4, 3) == want


def test_clock_matches_set_definition_bruteforce():
    # Alg. 1: clock k = {(i,j): 1<=i<=m, 1<=j<=n, i+j-1 = k}, k = 1..m+n-1
    for m, n in itertools.product(range(1, 9), range(1, 9)):
        allt = []
        for k in range(1, m + n):
            want = {(i, j) for i in range(1, m + 1) for j in range(1, n + 1) if i + j - 1 == k}
            got = S.clock(k, m, n)
            assert set(got) == want and len(got) == len(want)
            assert [j for _, j in got] == sorted(j for _, j in got)
            allt += got
        assert len(allt) == m * n and len(set(allt)) == m * n  # every task exactly once
        assert S.clock(m + n, m, n) == []


def test_device_order_golden_fig1_case():
    g = _parse_golden("device_order_m4_n3_except_last.txt")
    recs = S.records(4, 3, "except_last")
    names = {S.F: "F", S.RECOMPUTE: "R", S.B: "B"}
    for j in (1, 2, 3):
        got = []
        for kind, i in S.device_order(recs, j):
            got.append(f"W{j}" if kind == S.W else f"{names[kind]}{i}{j}")
        assert got == g[j]


@pytest.mark.parametrize("mode,per_dev", [("always", lambda m: m), ("except_last", lambda m: m - 1),
                                          ("never", lambda m: 0)])
def test_recompute_counts(mode, per_dev):
    # P:105 F' for every B; P:108 F'_m omitted; m = 1 under except_last => none (P:305 footnote)
    for m, n in itertools.product(range(1, 7), range(1, 5)):
        recs = S.records(m, n, mode)
        for j in range(1, n + 1):
            cnt = sum(1 for r in recs if r[2] == S.RECOMPUTE and r[4] == j)
            assert cnt == per_dev(m)


def test_per_device_order_invariants():
    # F_{i,j} before F_{i+1,j}; B_{i,j} before B_{i-1,j}; F'_{i,j} right before B_{i,j}
    for m, n, mode in itertools.product(range(1, 7), range(1, 5), S.MODES):
        recs = S.records(m, n, mode)
        for j in range(1, n + 1):
            od = S.device_order(recs, j)
            fs = [i for k, i in od if k == S.F]
            bs = [i for k, i in od if k == S.B]
            assert fs == list(range(1, m + 1))
            assert bs == list(range(m, 0, -1))
            for p, (k, i) in enumerate(od):
                if k == S.RECOMPUTE:
                    assert od[p + 1] == (S.B, i)
            assert od[-1] == (S.W, 0)
            assert od.index((S.B, m)) > od.index((S.F, m))


def test_copies_precede_computes_within_clock():
    # Alg. 1: in clock k all copies are issued first, then the computes
    recs = S.records(5, 4, "except_last", routes=[(1, 4), (2, 3)])
    for ph in (0, 1):
        for k in range(1, 9):
            kinds = [r[2] for r in recs if r[0] == ph and r[1] == k]
            first_compute = next(p for p, kk in enumerate(kinds) if kk in (S.F, S.RECOMPUTE, S.B))
            assert all(kk in (S.F, S.RECOMPUTE, S.B) for kk in kinds[first_compute:])


def test_record_counts_c4_routes():
    # SURVEY Appendix A.3 counts at (m=32, n=8, always) with the C4 routes
    routes = [(1, 7), (2, 6), (3, 5), (3, 4)]
    recs = S.records(32, 8, "always", routes)
    cnt = {k: int((recs[:, 2] == k).sum()) for k in range(8)}
    assert cnt == {S.F: 256, S.RECOMPUTE: 256, S.B: 256, S.COPY_F: 224, S.COPY_B: 224,
                   S.SKIP_F: 128, S.SKIP_B: 128, S.W: 8}
    recs = S.records(32, 8, "except_last")
    assert int((recs[:, 2] == S.RECOMPUTE).sum()) == 248
    # clocks: m + n - 1 per phase
    assert recs[recs[:, 0] == 0][:, 1].max() == 39 and recs[recs[:, 0] == 1][:, 1].max() == 39


def test_skip_same_partition_has_no_copy():
    recs = S.records(4, 3, "never", routes=[(2, 2), (1, 3)])
    assert not any(r[7] == 0 for r in recs if r[2] in (S.SKIP_F, S.SKIP_B))
    assert sum(1 for r in recs if r[2] == S.SKIP_F) == 4
    # portals: one hop s -> d regardless of distance (Fig. 6 caption P:221), vs d - s hops tuple-threaded
    recs = S.records(1, 4, "never", routes=[(1, 4)])
    sk = [r for r in recs if r[2] == S.SKIP_F]
    assert len(sk) == 1 and (sk[0][5], sk[0][6]) == (1, 4)


def _list_schedule_makespan(m, n, cost=1.0):
    """Unit-cost event simulation of the forward tasks: device j runs its F tasks in order, each
    starting when both the device is free and F_{i,j-1} finished (copy cost 0)."""
    recs = S.records(m, n, "never")
    done = {}
    free = [0.0] * (n + 1)
    for r in recs:
        if r[0] != 0 or r[2] != S.F:
            continue
        i, j = int(r[3]), int(r[4])
        start = max(free[j], done.get((i, j - 1), 0.0))
        done[(i, j)] = start + cost
        free[j] = start + cost
    return max(done.values())


def test_forward_makespan_closed_form():
    # SPEC S:265 / acceptance 5: forward makespan (m+n-1) c; busy fraction m/(m+n-1)
    for m, n in itertools.product(range(1, 7), range(1, 7)):
        assert _list_schedule_makespan(m, n, 2.0) == 2.0 * (m + n - 1)


def test_split_sizes():
    # SPEC S:326-327 examples (reading Z7)
    assert S.split_sizes(8, 4) == [2, 2, 2, 2]
    assert S.split_sizes(10, 4) == [3, 3, 2, 2]
    assert S.split_sizes(512, 32) == [16] * 32
    with pytest.raises(ValueError):
        S.split_sizes(3, 4)
    x = np.arange(30).reshape(10, 3)
    off = S.split_offsets(10, 4)
    assert np.array_equal(np.concatenate([x[off[i]:off[i + 1]] for i in range(4)]), x)
