"""Philox4x32-10 counter-based RNG and the dropout rule (reading Z17)
-- TEST INFRASTRUCTURE ONLY.

The paper asks only that recomputation be "referentially transparent" (P:122 footnote) and
that checkpointed stages recompute "under the restored RNG state" (BASELINE.json north star).
With a counter-based generator keyed by the global element index, the "saved RNG state" is
just (seed, step): recomputation F' reproduces every mask bit-exactly and the pipelined run
equals the full-batch run even with dropout.

Philox4x32-10 (Salmon et al., SC'11):  round(c, k):
  (hi0, lo0) = mulhilo(0xD2511F53, c0);  (hi1, lo1) = mulhilo(0xCD9E8D57, c2)
  c' = (hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0)
  k' = (k0 + 0x9E3779B9, k1 + 0xBB67AE85)
ten rounds, the key bumped between rounds.
"""
import numpy as np

M0, M1 = 0xD2511F53, 0xCD9E8D57
W0, W1 = 0x9E3779B9, 0xBB67AE85
MASK = 0xFFFFFFFF


def philox4x32_10(ctr, key):
    """Scalar reference: ctr = 4 ints, key = 2 ints -> 4 ints (Python big ints, obviously exact)."""
    c0, c1, c2, c3 = [int(v) & MASK for v in ctr]
    k0, k1 = [int(v) & MASK for v in key]
    for r in range(10):
        p0 = M0 * c0
        p1 = M1 * c2
        hi0, lo0 = p0 >> 32, p0 & MASK
        hi1, lo1 = p1 >> 32, p1 & MASK
        c0, c1, c2, c3 = (hi1 ^ c1 ^ k0) & MASK, lo1, (hi0 ^ c3 ^ k1) & MASK, lo0
        if r < 9:
            k0, k1 = (k0 + W0) & MASK, (k1 + W1) & MASK
    return (c0, c1, c2, c3)


def philox_vec(c0, c1, c2, c3, k0, k1):
    """Vectorised numpy version over uint64 arrays holding 32-bit values (same rounds)."""
    c0, c1, c2, c3 = [np.asarray(v, dtype=np.uint64) & MASK for v in (c0, c1, c2, c3)]
    k0 = np.uint64(int(k0) & MASK)
    k1 = np.uint64(int(k1) & MASK)
    m0, m1 = np.uint64(M0), np.uint64(M1)
    for r in range(10):
        p0 = m0 * c0
        p1 = m1 * c2
        hi0, lo0 = p0 >> np.uint64(32), p0 & np.uint64(MASK)
        hi1, lo1 = p1 >> np.uint64(32), p1 & np.uint64(MASK)
        c0, c1, c2, c3 = (hi1 ^ c1 ^ k0), lo1, (hi0 ^ c3 ^ k1), lo0
        if r < 9:
            k0 = (k0 + np.uint64(W0)) & np.uint64(MASK)
            k1 = (k1 + np.uint64(W1)) & np.uint64(MASK)
    return c0, c1, c2, c3


def dropout_keep(seed, step, site, row0, rows, cols, p):
    """Keep-mask for a [rows, cols] block whose first row is global row `row0` of a
    row-major [B, cols] tensor (O8):
        idx = global flat index, q = idx >> 2,
        ctr = (q_lo, q_hi, site, step), key = (seed_lo, seed_hi),
        word = philox(ctr, key)[idx & 3],  u = (word >> 8) * 2^-24,  keep iff u >= p.
    """
    r = np.arange(row0, row0 + rows, dtype=np.uint64)[:, None]
    c = np.arange(cols, dtype=np.uint64)[None, :]
    idx = r * np.uint64(cols) + c
    q = idx >> np.uint64(2)
    w = philox_vec(q & np.uint64(MASK), q >> np.uint64(32), np.full_like(q, site),
                   np.full_like(q, step), int(seed) & MASK, (int(seed) >> 32) & MASK)
    sel = (idx & np.uint64(3)).astype(np.int64)
    word = np.choose(sel, w)
    u = (word >> np.uint64(8)).astype(np.float64) * 2.0 ** -24
    return u >= p
