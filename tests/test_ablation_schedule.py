"""Host logic of the Table 1 ablation schedules, through the
C ABI's pure host entry point tgp_schedule_ablation (no GPU).  The oracle has no counterpart for
these orders (they are the paper's *baselines*, not its method), so they are pinned by the
properties that define them: the same task multiset as the method's schedule, a topological order
of the backward dependencies (so issue can never deadlock), and the hop structure of a
tuple-threaded skip tensor (carried through every partition in between)."""
import numpy as np
import pytest

from oracle.schedule import records, route_partitions
from synth import configs as C

tgp = pytest.importorskip("paper_2004_09910_b200.tgp")

F, RECOMPUTE, B, COPY_F, COPY_B, SKIP_F, SKIP_B, W = range(8)

UMLP = C.umlp(d=64)
BAL = [2, 3, 3, 3, 3, 3, 3, 3]
ROUTES = route_partitions(UMLP, BAL)  # 1-based (src, dst) partition pairs


@pytest.mark.parametrize("m,n,mode", [(4, 8, "except_last"), (3, 2, "always"), (5, 3, "never")])
def test_no_toggles_is_the_method_schedule(m, n, mode):
    routes = ROUTES if n == 8 else [(1, n)]
    a = tgp.schedule(m, n, mode, routes)
    b = tgp.schedule(m, n, mode, routes, relay=False, order_seed=0)
    assert np.array_equal(a, b)
    assert np.array_equal(a, records(m, n, mode, routes))


def test_relay_hops_follow_the_activation():
    m, n = 4, 8
    portal = tgp.schedule(m, n, "except_last", ROUTES)
    relay = tgp.schedule(m, n, "except_last", ROUTES, relay=True)
    # everything but the skip records is unchanged, in the same order
    keep = lambda r: r[~np.isin(r[:, 2], [SKIP_F, SKIP_B])]
    assert np.array_equal(keep(portal), keep(relay))
    pos = {tuple(r[[0, 2, 3, 4]]): k for k, r in enumerate(relay) if r[2] in (F, B)}
    for q, (s, d) in enumerate(ROUTES):
        for i in range(1, m + 1):
            f = relay[(relay[:, 2] == SKIP_F) & (relay[:, 7] == q) & (relay[:, 3] == i)]
            assert [tuple(x) for x in f[:, 5:7]] == [(j - 1, j) for j in range(s + 1, d + 1)]
            for rec in f:  # each hop is in F_{i,j}'s clock, before F_{i,j}
                k = [k for k, r in enumerate(relay) if (r == rec).all()][0]
                assert relay[pos[(0, F, i, rec[6])]][1] == rec[1] and k < pos[(0, F, i, rec[6])]
            b = relay[(relay[:, 2] == SKIP_B) & (relay[:, 7] == q) & (relay[:, 3] == i)]
            assert [tuple(x) for x in b[:, 5:7]] == [(j + 1, j) for j in range(d - 1, s - 1, -1)]
            for rec in b:
                k = [k for k, r in enumerate(relay) if (r == rec).all()][0]
                assert relay[pos[(1, B, i, rec[6])]][1] == rec[1] and k < pos[(1, B, i, rec[6])]
    # a tuple-threaded skip costs (d - s) copies per micro-batch and direction, a portal one
    n_portal = int(np.isin(portal[:, 2], [SKIP_F, SKIP_B]).sum())
    n_relay = int(np.isin(relay[:, 2], [SKIP_F, SKIP_B]).sum())
    assert n_portal == 2 * m * len(ROUTES)
    assert n_relay == 2 * m * sum(d - s for s, d in ROUTES) > n_portal


def test_relay_of_adjacent_route_equals_portal():
    a = tgp.schedule(4, 3, "except_last", [(1, 2), (2, 3)])
    b = tgp.schedule(4, 3, "except_last", [(1, 2), (2, 3)], relay=True)
    assert np.array_equal(a, b)


def _check_topological(bw, m, n, routes, mode, relay):
    done_b = set()
    seen_copy = set()
    arrived = {}
    for k, r in enumerate(bw):
        kind, i, j, src, dst, q = r[2], r[3], r[4], r[5], r[6], r[7]
        if kind == COPY_B:
            assert (i, src) in done_b, f"COPY_B({i},{src}->{dst}) before B_{i},{src}"
            seen_copy.add((i, dst))
        elif kind == SKIP_B:
            assert (i, src) in done_b, f"SKIP_B hop {src}->{dst} before B_{i},{src}"
            arrived.setdefault((i, dst), set()).add(q)
        elif kind == RECOMPUTE:
            nxt = bw[k + 1]
            assert nxt[2] == B and nxt[3] == i and nxt[4] == j  # F' right before its B
        elif kind == B:
            assert (i, j) not in done_b
            if j < n:
                assert (i, j + 1) in done_b and (i, j) in seen_copy
            for q2, (s, d) in enumerate(routes):
                if s == d:
                    continue
                if (s == j) or (relay and s < j < d):
                    assert q2 in arrived.get((i, j), set()), f"B_{i},{j} before its skip gradient"
            done_b.add((i, j))
    assert len(done_b) == m * n


@pytest.mark.parametrize("seed", [1, 2, 12345])
@pytest.mark.parametrize("relay", [False, True])
def test_unordered_backward_is_a_topological_permutation(seed, relay):
    m, n, mode = 4, 8, "except_last"
    ordered = tgp.schedule(m, n, mode, ROUTES, relay=relay)
    un = tgp.schedule(m, n, mode, ROUTES, relay=relay, order_seed=seed)
    # forward and W records untouched
    assert np.array_equal(ordered[ordered[:, 0] != 1], un[un[:, 0] != 1])
    key = lambda r: sorted(tuple(x) for x in r[r[:, 0] == 1][:, 2:])
    assert key(ordered) == key(un)  # same backward tasks and messages
    bw = un[un[:, 0] == 1]
    _check_topological(bw, m, n, ROUTES, mode, relay)
    _check_topological(ordered[ordered[:, 0] == 1], m, n, ROUTES, mode, relay)
    # deterministic per seed; the step (clock) field counts issue steps 1..m*n
    assert np.array_equal(un, tgp.schedule(m, n, mode, ROUTES, relay=relay, order_seed=seed))
    assert sorted(set(bw[:, 1].tolist())) == list(range(1, m * n + 1))


def test_unordered_backward_breaks_the_fork_join_order():
    # with the Fork/Join edge every device runs B in descending i; a random
    # topological order does not, on at least one device, and differs across seeds
    m, n = 8, 4
    orders = []
    for seed in (1, 2, 3):
        bw = tgp.schedule(m, n, "never", [], order_seed=seed)
        bw = bw[(bw[:, 0] == 1) & (bw[:, 2] == B)]
        per_dev = {j: bw[bw[:, 4] == j][:, 3].tolist() for j in range(1, n + 1)}
        assert any(v != sorted(v, reverse=True) for v in per_dev.values())
        orders.append(per_dev)
    assert orders[0] != orders[1] or orders[1] != orders[2]
    ref = tgp.schedule(m, n, "never", [])
    ref = ref[(ref[:, 0] == 1) & (ref[:, 2] == B)]
    for j in range(1, n + 1):
        assert ref[ref[:, 4] == j][:, 3].tolist() == list(range(m, 0, -1))
