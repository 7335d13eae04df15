"""Pins for oracle encode/decode (O5): exact high-precision canonical-embedding sums
(mpmath), round trip, constant -> constant polynomial."""
import mpmath
import numpy as np
import pytest

from oracle import encoding


def _encode_mp(z, n, scale):
    """O5 by definition in 60-digit arithmetic: m_k = round((2/N) Re sum_j z_j zeta^{-5^j k} * scale)."""
    mpmath.mp.dps = 60
    out = []
    for k in range(n):
        acc = mpmath.mpf(0)
        x = 1
        for j in range(n // 2):
            zj = z[j] if j < len(z) else 0.0
            acc += mpmath.mpf(zj) * mpmath.cos(-mpmath.pi * ((x * k) % (2 * n)) / n)
            x = x * 5 % (2 * n)
        out.append(int(mpmath.nint(2 * acc / n * mpmath.mpf(scale))))
    return out


@pytest.mark.parametrize("n", [16, 64])
def test_encode_matches_exact_definition(n):
    rng = np.random.default_rng(n)
    z = rng.uniform(-1, 1, n // 2)
    want = _encode_mp(z, n, 2.0 ** 40)
    got = encoding.encode(z, n, 2.0 ** 40)
    direct = encoding.encode_direct(z, n, 2.0 ** 40)
    assert np.max(np.abs(np.array(want) - got)) <= 1
    assert np.max(np.abs(np.array(want) - direct)) <= 1


@pytest.mark.parametrize("n", [8192, 16384])
def test_round_trip(n):
    rng = np.random.default_rng(1)
    z = rng.uniform(0, 1, n // 2)
    m = encoding.encode(z, n, 2.0 ** 40)
    back = encoding.decode(m, n, 2.0 ** 40, n // 2)
    assert np.max(np.abs(back - z)) < 2.0 ** -30


def test_decode_matches_direct():
    n = 64
    rng = np.random.default_rng(3)
    m = rng.integers(-2 ** 40, 2 ** 40, n)
    assert np.allclose(encoding.decode(m, n, 2.0 ** 40, n // 2), encoding.decode_direct(m, n, 2.0 ** 40, n // 2),
                       atol=1e-12)


@pytest.mark.parametrize("c", [0.5, -0.004, 0.197, 1.0])
def test_constant_encodes_to_constant_poly(c):
    n = 8192
    m = encoding.encode(np.full(n // 2, c), n, 2.0 ** 40)
    assert m[0] == int(np.rint(c * 2.0 ** 40))
    assert np.all(m[1:] == 0)


def test_partial_slots_zero_padded():
    n = 64
    z = np.array([0.25, 0.5, 0.75])
    m = encoding.encode(z, n, 2.0 ** 40)
    back = encoding.decode(m, n, 2.0 ** 40, n // 2)
    assert np.allclose(back[:3], z, atol=1e-9) and np.allclose(back[3:], 0, atol=1e-9)
