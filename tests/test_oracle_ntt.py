"""Pins for the oracle NTT (O3): O(N^2) definition, negacyclic convolution theorem,
round trip, closed forms for X^0 and X^1."""
import numpy as np
import pytest

from oracle import params, ring
from synth import random_residues


def _prime_and_psi(n, bits):
    p = params.select_primes([bits], n)[0]
    return p, params.minimal_psi(p, n)


@pytest.mark.parametrize("n", [8, 16, 64, 256])
@pytest.mark.parametrize("bits", [40, 60])
def test_ntt_matches_definition(n, bits):
    q, psi = _prime_and_psi(n, bits)
    a = random_residues((3, n), [q] * 3, seed=n + bits)
    got = ring.ntt_fwd(a, [q] * 3, [psi] * 3)
    for r in range(3):
        assert [int(v) for v in got[r]] == ring.ntt_definition(a[r].tolist(), q, psi)


def _schoolbook_negacyclic(a, b, q):
    n = len(a)
    out = [0] * n
    for i in range(n):
        ai = int(a[i])
        for j in range(n):
            k = i + j
            if k < n:
                out[k] += ai * int(b[j])
            else:
                out[k - n] -= ai * int(b[j])
    return [v % q for v in out]


@pytest.mark.parametrize("n", [16, 128, 1024])
def test_negacyclic_convolution_theorem(n):
    q, psi = _prime_and_psi(n, 60)
    a = random_residues((1, n), [q], seed=1)[0]
    b = random_residues((1, n), [q], seed=2)[0]
    A = ring.ntt_fwd(a[None], [q], [psi])[0]
    B = ring.ntt_fwd(b[None], [q], [psi])[0]
    c = ring.ntt_inv(ring.mul(A, B, q)[None], [q], [psi])[0]
    assert [int(v) for v in c] == _schoolbook_negacyclic(a, b, q)


@pytest.mark.parametrize("depth", [2, 4])
def test_round_trip_full_size(depth):
    pr = params.params_from_depth(depth)
    qs, ps = pr.moduli, pr.psi
    a = random_residues((len(qs), pr.n), qs, seed=7)
    A = ring.ntt_fwd(a, qs, ps)
    assert not np.array_equal(A, a)
    assert np.array_equal(ring.ntt_inv(A, qs, ps), a)


def test_closed_forms_monomials():
    n = 4096
    q, psi = _prime_and_psi(n, 40)
    logn = n.bit_length() - 1
    one = np.zeros(n, dtype=np.uint64); one[0] = 1
    assert np.all(ring.ntt_fwd(one[None], [q], [psi])[0] == 1)
    x = np.zeros(n, dtype=np.uint64); x[1] = 1
    got = ring.ntt_fwd(x[None], [q], [psi])[0]
    want = [pow(psi, 2 * ring.bitrev(k, logn) + 1, q) for k in range(n)]
    assert [int(v) for v in got] == want


def test_elementwise_against_python_ints():
    q = params.params_from_depth(4).q[0]
    rng = np.random.default_rng(5)
    a = rng.integers(0, q, 1000, dtype=np.uint64)
    b = rng.integers(0, q, 1000, dtype=np.uint64)
    ai, bi = [int(v) for v in a], [int(v) for v in b]
    assert [int(v) for v in ring.mul(a, b, q)] == [x * y % q for x, y in zip(ai, bi)]
    assert [int(v) for v in ring.add(a, b, q)] == [(x + y) % q for x, y in zip(ai, bi)]
    assert [int(v) for v in ring.sub(a, b, q)] == [(x - y) % q for x, y in zip(ai, bi)]
    q2 = params.params_from_depth(4).q[1]
    assert [int(v) for v in ring.center_mod(a, q, q2)] == [((x - q) if x > (q - 1) // 2 else x) % q2 for x in ai]
    assert [int(v) for v in ring.reduce(a, q2)] == [x % q2 for x in ai]
