"""Philox4x32-10 counter-based generator (Salmon et al., SC'11), vectorised in numpy.

This module holds NO arithmetic of the EFGP method: it only turns (seed, stream, record, k)
into pseudo-random doubles.  It is shared by the tests, the bench and (through the identical CUDA
implementation in ``efgp_data/csrc/efgp_datagen.cu``) the device-side generator used for N = 1e9.

Layout (our reading G7 of BASELINE.json, which names seeds but no generator):
  key = (seed, 0); double #k of record n in stream s comes from counter (n_lo, s, k // 2, n_hi),
  words (2 (k mod 2), 2 (k mod 2) + 1) -> u = (hi * 2^21 + (lo >> 11)) * 2^-53 in [0, 1).
"""
from __future__ import annotations

import numpy as np

M0 = np.uint64(0xD2511F53)
M1 = np.uint64(0xCD9E8D57)
W0 = np.uint32(0x9E3779B9)
W1 = np.uint32(0xBB67AE85)
MASK32 = np.uint64(0xFFFFFFFF)

STREAM_POINTS = 0
STREAM_NOISE = 1
STREAM_TARGETS = 2
STREAM_COMPONENT = 3


def philox4x32_10(c0, c1, c2, c3, k0, k1):
    """Ten Philox4x32 rounds.  All inputs uint32 arrays (broadcastable); returns 4 uint32 arrays."""
    c0 = np.asarray(c0, dtype=np.uint32).astype(np.uint64)
    c1 = np.asarray(c1, dtype=np.uint32).astype(np.uint64)
    c2 = np.asarray(c2, dtype=np.uint32).astype(np.uint64)
    c3 = np.asarray(c3, dtype=np.uint32).astype(np.uint64)
    k0 = np.uint32(k0)
    k1 = np.uint32(k1)
    c0, c1, c2, c3 = np.broadcast_arrays(c0, c1, c2, c3)
    for r in range(10):
        if r > 0:
            k0 = np.uint32((int(k0) + int(W0)) & 0xFFFFFFFF)
            k1 = np.uint32((int(k1) + int(W1)) & 0xFFFFFFFF)
        p0 = M0 * c0
        p1 = M1 * c2
        hi0, lo0 = p0 >> np.uint64(32), p0 & MASK32
        hi1, lo1 = p1 >> np.uint64(32), p1 & MASK32
        c0, c1, c2, c3 = (hi1 ^ c1 ^ np.uint64(k0)), lo1, (hi0 ^ c3 ^ np.uint64(k1)), lo0
    return tuple(a.astype(np.uint32) for a in (c0, c1, c2, c3))


def uniform(seed: int, stream: int, records, k: int) -> np.ndarray:
    """Double #k in [0, 1) of each record index in `records` for the given stream."""
    n = np.asarray(records, dtype=np.uint64)
    w = philox4x32_10((n & MASK32).astype(np.uint32), np.uint32(stream), np.uint32(k // 2),
                      (n >> np.uint64(32)).astype(np.uint32), np.uint32(seed & 0xFFFFFFFF), np.uint32(0))
    hi = w[2 * (k % 2)].astype(np.uint64)
    lo = w[2 * (k % 2) + 1].astype(np.uint64)
    return ((hi << np.uint64(21)) + (lo >> np.uint64(11))).astype(np.float64) * 2.0 ** -53


def normal(seed: int, stream: int, records, k: int) -> np.ndarray:
    """Standard normal from doubles (k, k+1) by Box-Muller's cos branch:
    sqrt(-2 log(1 - u1)) cos(2 pi u2)  (1 - u1 in (0, 1] keeps the log finite)."""
    u1 = uniform(seed, stream, records, k)
    u2 = uniform(seed, stream, records, k + 1)
    return np.sqrt(-2.0 * np.log1p(-u1)) * np.cos(2.0 * np.pi * u2)
