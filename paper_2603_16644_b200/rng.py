"""Deterministic random streams (host side), identical to src/rng.py:23-46.

The sketch operator's signs and sampled rows are a function of (m, d, transform,
seed) through numpy's Philox keyed by `seed | lane << 64`; keeping the same
generator makes our operators bitwise equal to the reference's, which is what
the "exact-S oracle mode" parity gate requires.
"""

import hashlib

import numpy as np

MASK64 = (1 << 64) - 1
LANE_SKETCH_SIGNS = 1
LANE_SKETCH_ROWS = 2
LANE_GAUSSIAN = 3


def stream(seed, lane=0):
    """Generator for sub-stream `lane` of `seed` (Philox key = seed | lane << 64)."""
    return np.random.Generator(np.random.Philox(
        key=(int(seed) & MASK64) | ((int(lane) & MASK64) << 64)))


def mix64(*parts):
    """blake2b-8 hash of 16-byte little-endian signed integers -> 64-bit seed."""
    h = hashlib.blake2b(digest_size=8)
    for p in parts:
        h.update(int(p).to_bytes(16, "little", signed=True))
    return int.from_bytes(h.digest(), "little")
