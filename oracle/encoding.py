"""Oracle: CKKS canonical-embedding encode/decode (TEST INFRASTRUCTURE ONLY).

Background the paper relies on ("a sequence of values ... encoded into a single
polynomial") but does not print.  Slots n = N/2; slot j <-> the root
zeta^{5^j mod 2N}, zeta = exp(i pi / N).

    encode:  u_k = (2/N) Re( sum_j z_j zeta^{-5^j k} ),  m_k = rint(Delta * u_k)
    decode:  z_j = Re( sum_k m_k zeta^{5^j k} ) / scale

``encode_direct``/``decode_direct`` are these sums written out (O(N*n)); the FFT
forms use numpy's FFT as a library step (m(zeta^{2t+1}) = sum_k (m_k zeta^k) w^{tk},
w = zeta^2) and are pinned against the direct forms in the tests.
"""
from __future__ import annotations

import numpy as np


def _slot_positions(n_poly: int) -> np.ndarray:
    """t_j with 2 t_j + 1 = 5^j mod 2N, for j < N/2."""
    two_n = 2 * n_poly
    e = np.empty(n_poly // 2, dtype=np.int64)
    x = 1
    for j in range(n_poly // 2):
        e[j] = x
        x = x * 5 % two_n
    return e


def encode_direct(z, n_poly: int, scale: float) -> np.ndarray:
    z = np.asarray(z, dtype=np.float64)
    n_slots = n_poly // 2
    zz = np.zeros(n_slots, dtype=np.complex128)
    zz[: z.size] = z
    e = _slot_positions(n_poly)
    k = np.arange(n_poly)
    # zeta^{-5^j k} = exp(-i pi 5^j k / N); exponent reduced mod 2N exactly in integers
    out = np.empty(n_poly, dtype=np.int64)
    for kk in range(n_poly):
        ang = -np.pi * ((e * kk) % (2 * n_poly)) / n_poly
        u = 2.0 / n_poly * np.real(np.sum(zz * np.exp(1j * ang)))
        out[kk] = np.int64(np.rint(scale * u))
    del k
    return out


def encode(z, n_poly: int, scale: float) -> np.ndarray:
    """FFT form of O5; returns int64 coefficients m_k = rint(scale * u_k)."""
    z = np.asarray(z, dtype=np.float64)
    n_slots = n_poly // 2
    if z.size > n_slots:
        raise ValueError("CapacityError: more values than slots")
    e = _slot_positions(n_poly)
    v = np.zeros(n_poly, dtype=np.complex128)
    zz = np.zeros(n_slots, dtype=np.complex128)
    zz[: z.size] = z
    v[(e - 1) // 2] = zz
    v[(2 * n_poly - e - 1) // 2] = np.conj(zz)
    w = np.fft.fft(v) / n_poly                       # w_k = m_k zeta^k
    k = np.arange(n_poly)
    u = np.real(w * np.exp(-1j * np.pi * k / n_poly))
    return np.rint(scale * u).astype(np.int64)


def decode_direct(m, n_poly: int, scale: float, n_out: int) -> np.ndarray:
    m = np.asarray(m, dtype=np.float64)
    e = _slot_positions(n_poly)
    k = np.arange(n_poly)
    out = np.empty(n_out)
    for j in range(n_out):
        ang = np.pi * ((int(e[j]) * k) % (2 * n_poly)) / n_poly
        out[j] = np.real(np.sum(m * np.exp(1j * ang))) / scale
    return out


def decode(m, n_poly: int, scale: float, n_out: int) -> np.ndarray:
    """FFT form: v_t = sum_k (m_k zeta^k) w^{tk} = N ifft(m zeta^k)[t]; z_j = Re v_{t_j} / scale."""
    m = np.asarray(m, dtype=np.float64)
    k = np.arange(n_poly)
    v = np.fft.ifft(m * np.exp(1j * np.pi * k / n_poly)) * n_poly
    e = _slot_positions(n_poly)
    return np.real(v[(e[:n_out] - 1) // 2]) / scale
