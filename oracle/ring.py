"""Oracle: RNS polynomial-ring helpers over numpy uint64 (TEST INFRASTRUCTURE ONLY).

Thin wrappers over oracle/ring_oracle.c; every row of an array is one limb (one
polynomial modulo one prime).  The O(N^2) definition of the NTT (O3) lives here in
pure Python integers and pins the fast C transform in the tests.
"""
from __future__ import annotations

import numpy as np

from ._lib import lib


def _rows(a: np.ndarray) -> np.ndarray:
    return a.reshape(-1, a.shape[-1])


def ntt_fwd(a: np.ndarray, moduli, psis) -> np.ndarray:
    """Forward negacyclic NTT of each row; ``moduli``/``psis`` are per row (len = rows)."""
    x = np.ascontiguousarray(a, dtype=np.uint64).copy()
    r = _rows(x)
    q = np.ascontiguousarray(np.asarray(moduli, dtype=np.uint64).reshape(-1))
    p = np.ascontiguousarray(np.asarray(psis, dtype=np.uint64).reshape(-1))
    assert q.size == r.shape[0] and p.size == r.shape[0]
    scratch = np.zeros(r.shape[1], dtype=np.uint64)
    lib().orc_ntt_fwd(r, r.shape[0], r.shape[1], q, p, scratch)
    return x


def ntt_inv(a: np.ndarray, moduli, psis) -> np.ndarray:
    x = np.ascontiguousarray(a, dtype=np.uint64).copy()
    r = _rows(x)
    q = np.ascontiguousarray(np.asarray(moduli, dtype=np.uint64).reshape(-1))
    p = np.ascontiguousarray(np.asarray(psis, dtype=np.uint64).reshape(-1))
    assert q.size == r.shape[0] and p.size == r.shape[0]
    scratch = np.zeros(r.shape[1], dtype=np.uint64)
    lib().orc_ntt_inv(r, r.shape[0], r.shape[1], q, p, scratch)
    return x


def bitrev(k: int, bits: int) -> int:
    r = 0
    for _ in range(bits):
        r = (r << 1) | (k & 1)
        k >>= 1
    return r


def ntt_definition(a, q: int, psi: int):
    """O3 by definition, O(N^2) Python ints: A[k] = sum_j a_j psi^{(2 brv(k)+1) j} mod q."""
    n = len(a)
    logn = n.bit_length() - 1
    out = []
    for k in range(n):
        e = 2 * bitrev(k, logn) + 1
        w = pow(psi, e, q)
        acc, wj = 0, 1
        for j in range(n):
            acc += int(a[j]) * wj
            wj = wj * w % q
        out.append(acc % q)
    return out


def mul(a, b, q):
    out = np.empty_like(a)
    lib().orc_vec_mul(out, np.ascontiguousarray(a), np.ascontiguousarray(b), a.size, q)
    return out


def mul_scalar(a, s, q):
    out = np.empty_like(a)
    lib().orc_vec_mul_scalar(out, np.ascontiguousarray(a), int(s) % q, a.size, q)
    return out


def add(a, b, q):
    out = np.empty_like(a)
    lib().orc_vec_add(out, np.ascontiguousarray(a), np.ascontiguousarray(b), a.size, q)
    return out


def sub(a, b, q):
    out = np.empty_like(a)
    lib().orc_vec_sub(out, np.ascontiguousarray(a), np.ascontiguousarray(b), a.size, q)
    return out


def add_scalar(a, s, q):
    out = np.empty_like(a)
    lib().orc_vec_add_scalar(out, np.ascontiguousarray(a), int(s) % q, a.size, q)
    return out


def reduce(a, q):
    """a mod q for arbitrary uint64 (plain unsigned reduction)."""
    out = np.empty_like(a)
    lib().orc_vec_mod(out, np.ascontiguousarray(a), a.size, q)
    return out


def from_signed(a, q):
    out = np.empty(a.shape, dtype=np.uint64)
    lib().orc_vec_from_signed(out, np.ascontiguousarray(a, dtype=np.int64), a.size, q)
    return out


def center_mod(r, q_from, q_to):
    """Centered lift of r in [0,q_from) to (-q_from/2, q_from/2], reduced mod q_to."""
    out = np.empty_like(r)
    lib().orc_vec_center_mod(out, np.ascontiguousarray(r), r.size, q_from, q_to)
    return out


def inv(a: int, q: int) -> int:
    return pow(a, q - 2, q)
