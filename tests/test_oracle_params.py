"""Pins for oracle/params.py: Alg. 8 hand traces, prime rule O2, root rule O3."""
import json
import os

import pytest

from oracle import params

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_alg8_hand_traces():
    cases = json.load(open(os.path.join(GOLD, "alg8_traces.json")))["cases"]
    for c in cases:
        d = params.parameterise(c["c"], c["s"], c["p"])
        assert d["coeff_mod_bits"] == c["coeff_mod_bits"], c
        assert d["poly_modulus_degree"] == c["poly_modulus_degree"], c
        assert d["scheme"] == 2 and d["scale"] == 2 ** c["s"]


@pytest.mark.parametrize("c", range(0, 12))
def test_alg8_properties(c):
    d = params.parameterise(c)
    m, n = d["coeff_mod_bits"], d["poly_modulus_degree"]
    assert len(m) == c + 2
    assert n % 1024 == 0 and (n // 1024) & (n // 1024 - 1) == 0    # 1024 * 2^k
    assert sum(m) <= 27 * n // 1024                                 # doubling bound
    assert n == 1024 or sum(m) > 27 * (n // 2) // 1024               # minimality of the doubling


def test_alg8_negative_cost():
    with pytest.raises(ValueError):
        params.parameterise(-1)


def _trial_division_prime(n):
    if n < 2:
        return False
    i = 2
    while i * i <= n:
        if n % i == 0:
            return False
        i += 1
    return True


def test_is_prime_small_vs_trial_division():
    for n in range(0, 5000):
        assert params.is_prime(n) == _trial_division_prime(n), n


def test_is_prime_known_values():
    assert params.is_prime(2 ** 61 - 1)            # Mersenne prime M61
    assert params.is_prime(2 ** 31 - 1)
    assert not params.is_prime(2 ** 59 - 1)        # 179951 * 3203431780337
    assert not params.is_prime(3215031751)         # strong pseudoprime to bases 2,3,5,7
    assert not params.is_prime(561) and not params.is_prime(41041)   # Carmichael numbers
    assert not params.is_prime(179951 * 3203431780337)


def _fermat_probable_prime(n):
    """Independent check (Fermat, several bases) -- a different test from Miller-Rabin."""
    return all(pow(a, n - 1, n) == 1 for a in (2, 3, 5, 7, 11, 13, 17, 19, 23))


@pytest.mark.parametrize("depth", [2, 4])
def test_prime_rule_O2(depth):
    d = params.parameterise(depth)
    n, bits = d["poly_modulus_degree"], d["coeff_mod_bits"]
    primes = params.select_primes(bits, n)
    assert len(set(primes)) == len(primes)
    used = set()
    for b, p in zip(bits, primes):
        assert p < 2 ** b and p > 2 ** (b - 1)
        assert (p - 1) % (2 * n) == 0
        assert _fermat_probable_prime(p)
        # no larger unused candidate below 2^b is prime
        cand = p + 2 * n
        while cand < 2 ** b:
            if cand not in used:
                assert not _fermat_probable_prime(cand), hex(cand)
            cand += 2 * n
        used.add(p)


def test_survey_prime_values():
    """The values SURVEY §8(c) O2 lists (computed there with sympy) follow from the rule."""
    p0 = params.params_from_depth(2)
    assert [hex(x) for x in p0.q] == ["0xfffffffffffc001", "0xfffffdc001", "0xfffff4c001"]
    assert hex(p0.p_special) == "0xffffffffffe8001"
    p1 = params.params_from_depth(4)
    assert [hex(x) for x in p1.q] == ["0xffffffffffe8001", "0xffffe80001", "0xffffca8001",
                                      "0xffffc40001", "0xffffb20001"]
    assert hex(p1.p_special) == "0xffffffffffd8001"


def _order(x, q):
    k, y = 1, x
    while y != 1:
        y = y * x % q
        k += 1
    return k


def test_minimal_psi_brute_force_tiny():
    # tiny NTT-friendly primes: brute force the minimal element of order exactly 2N
    for q, n in [(17, 8), (97, 16), (257, 64), (7681, 256), (12289, 512)]:
        want = min(x for x in range(2, q) if _order(x, q) == 2 * n)
        assert params.minimal_psi(q, n) == want


@pytest.mark.parametrize("depth", [2, 4])
def test_psi_is_primitive_2n_root(depth):
    pr = params.params_from_depth(depth)
    for q, psi in zip(pr.moduli, pr.psi):
        assert pow(psi, pr.n, q) == q - 1
        assert pow(psi, 2 * pr.n, q) == 1


def test_depth_chain_lengths():
    for c in (1, 2, 3, 4, 6):
        pr = params.params_from_depth(c)
        assert len(pr.q) == c + 1          # c rescales available (reading R1)
