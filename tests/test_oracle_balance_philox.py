"""Pins for oracle/balance.py (brute force) and oracle/philox.py (Random123 KATs)."""
import numpy as np
import pytest

from oracle import balance as Bal
from oracle import philox as Ph


def test_balance_examples():
    assert Bal.balance_dp([1, 2, 3, 4], 2) == [3, 1]            # SPEC S:440, max 6
    assert Bal.block_max([1, 2, 3, 4], [3, 1]) == 6
    assert Bal.balance_dp([5.0] * 32, 8) == [4] * 8             # uniform -> equal blocks
    assert Bal.balance_dp([7.0] * 4, 1) == [4]
    assert Bal.balance_dp([1, 1, 1], 3) == [1, 1, 1]
    with pytest.raises(ValueError):
        Bal.balance_dp([1, 2], 3)


def test_balance_vs_bruteforce_1000():
    rs = np.random.default_rng(7)
    for trial in range(1000):
        L = int(rs.integers(1, 13))
        n = int(rs.integers(1, min(4, L) + 1))
        if trial % 2:
            costs = [int(v) for v in rs.integers(0, 6, L)]   # many exact ties
        else:
            costs = [float(v) for v in rs.random(L)]
        dp = Bal.balance_dp(costs, n)
        bf = Bal.balance_brute(costs, n)
        assert sum(dp) == L and min(dp) >= 1 and len(dp) == n
        assert Bal.block_max(costs, dp) == pytest.approx(Bal.block_max(costs, bf), abs=1e-12)
        if trial % 2:
            assert dp == bf                                    # lexicographic tie-break on exact ties
        # scale invariance and monotonicity in n (SPEC balance invariants)
        assert Bal.balance_dp([4 * c for c in costs], n) == dp
        if n < L:
            assert Bal.block_max(costs, Bal.balance_dp(costs, n + 1)) <= Bal.block_max(costs, dp) + 1e-12


# Random123 known-answer vectors for philox4x32_10 (SURVEY §8(c) "O8 Philox" pin)
KAT = [
    ((0, 0, 0, 0), (0, 0), (0x6627e8d5, 0xe169c58d, 0xbc57ac4c, 0x9b00dbd8)),
    ((0xffffffff,) * 4, (0xffffffff,) * 2, (0x408f276d, 0x41c83b0e, 0xa20bc7c6, 0x6d5451fd)),
    ((0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344), (0xa4093822, 0x299f31d0),
     (0xd16cfe09, 0x94fdcceb, 0x5001e420, 0x24126ea1)),
]


@pytest.mark.parametrize("ctr,key,want", KAT)
def test_philox_kat(ctr, key, want):
    assert Ph.philox4x32_10(ctr, key) == want
    v = Ph.philox_vec(*[np.array([c], dtype=np.uint64) for c in ctr], *key)
    assert tuple(int(a[0]) for a in v) == want


def test_philox_vec_matches_scalar():
    rs = np.random.default_rng(3)
    c = rs.integers(0, 2 ** 32, size=(4, 64), dtype=np.uint64)
    k = [int(v) for v in rs.integers(0, 2 ** 32, size=2)]
    v = Ph.philox_vec(c[0], c[1], c[2], c[3], k[0], k[1])
    for t in range(64):
        assert tuple(int(a[t]) for a in v) == Ph.philox4x32_10([int(c[q, t]) for q in range(4)], k)


def test_dropout_keep_rate_and_global_index():
    p = 0.1
    keep = Ph.dropout_keep(1234, 5, 3, 0, 64, 1000, p)
    n = keep.size
    rate = keep.mean()
    assert abs(rate - (1 - p)) < 4 * np.sqrt(p * (1 - p) / n)
    # keyed by the GLOBAL element index: a sub-block equals the slice of the full mask
    sub = Ph.dropout_keep(1234, 5, 3, 16, 8, 1000, p)
    assert np.array_equal(sub, keep[16:24])
    # a different site / step / seed gives a different mask
    assert not np.array_equal(Ph.dropout_keep(1234, 5, 4, 0, 64, 1000, p), keep)
    assert not np.array_equal(Ph.dropout_keep(1234, 6, 3, 0, 64, 1000, p), keep)
    assert not np.array_equal(Ph.dropout_keep(1235, 5, 3, 0, 64, 1000, p), keep)
    # element idx uses word idx & 3 of philox(ctr = (idx >> 2, 0, site, step))
    w = Ph.philox4x32_10((1, 0, 3, 5), (1234, 0))
    idx = 6  # row 0 col 6 -> q = 1, word 2
    assert keep[0, 6] == ((w[2] >> 8) * 2.0 ** -24 >= p)
