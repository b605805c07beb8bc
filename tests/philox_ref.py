"""Test-side Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11 "Parallel random numbers: as easy as
1, 2, 3"), written in Python for the pins of the scenario draws (R3-R5).  It shares no
code with the oracle's C copy or the device copy; tests/test_oracle_draws.py checks it against the
Random123 known-answer vectors (tests/golden/philox_kat.txt) before using it.

The counter layout of one scenario draw is DESIGN.md's: ctr = (s, tag << 24 | c << 16, i, k >> 2),
key = (seed_lo, seed_hi), word k & 3; tags ARR 1, TIGHT 2, INST 3, KERN 4, SYNC 5, NOISE 6.
"""
M0, M1 = 0xD2511F53, 0xCD9E8D57
W0, W1 = 0x9E3779B9, 0xBB67AE85
MASK = 0xFFFFFFFF
TAG_ARR, TAG_TIGHT, TAG_INST, TAG_KERN, TAG_SYNC, TAG_NOISE = 1, 2, 3, 4, 5, 6


def philox4x32_10(ctr, key):
    c0, c1, c2, c3 = (int(x) & MASK for x in ctr)
    k0, k1 = (int(x) & MASK for x in key)
    for _ in range(10):
        p0, p1 = M0 * c0, M1 * c2
        c0, c1, c2, c3 = (p1 >> 32) ^ c1 ^ k0, p1 & MASK, (p0 >> 32) ^ c3 ^ k1, p0 & MASK
        k0, k1 = (k0 + W0) & MASK, (k1 + W1) & MASK
    return [c0, c1, c2, c3]


def word(seed, s, tag, c, i, k):
    out = philox4x32_10([s & MASK, (tag << 24) | (c << 16), i & MASK, k >> 2], [seed & MASK, (seed >> 32) & MASK])
    return out[k & 3]
