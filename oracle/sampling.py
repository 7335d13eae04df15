"""Oracle: seeded Philox4x32-10 samplers (TEST INFRASTRUCTURE ONLY).

Key (k0, k1) = (seed mod 2^32, seed >> 32); counter = (coefficient k, object id,
limb index, domain tag).  Domain tags below.  The GPU path implements the same
counter-based generator independently (reading Z10: CBD eta=21 errors instead of
SEAL's clipped Gaussian, so both sides are bit-exact).
"""
from __future__ import annotations

import numpy as np

from ._lib import lib

TAG_S, TAG_PK_A, TAG_PK_E, TAG_RLK_A, TAG_RLK_E, TAG_ENC_V, TAG_ENC_E0, TAG_ENC_E1 = 1, 2, 3, 4, 5, 6, 7, 8
TAG_GK_A, TAG_GK_E = 9, 10      # Galois keys (NEXT f1): object id = 64 * g + digit j
TAG_SK_A, TAG_SK_E = 11, 12     # secret-key encryption (wire compression, DESIGN reading Z16)


def philox4x32_10(ctr, key) -> np.ndarray:
    out = np.zeros(4, dtype=np.uint32)
    lib().orc_philox4x32_10(np.asarray(ctr, dtype=np.uint32), np.asarray(key, dtype=np.uint32), out)
    return out


def uniform(n: int, seed: int, obj: int, limb: int, tag: int, q: int) -> np.ndarray:
    out = np.zeros(n, dtype=np.uint64)
    lib().orc_sample_uniform(out, n, seed, obj, limb, tag, q)
    return out


def ternary(n: int, seed: int, obj: int, tag: int) -> np.ndarray:
    out = np.zeros(n, dtype=np.int64)
    lib().orc_sample_ternary(out, n, seed, obj, tag)
    return out


def cbd(n: int, seed: int, obj: int, tag: int) -> np.ndarray:
    out = np.zeros(n, dtype=np.int64)
    lib().orc_sample_cbd(out, n, seed, obj, tag)
    return out
