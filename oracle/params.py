"""Oracle: CKKS parameters (TEST INFRASTRUCTURE ONLY).

* ``parameterise`` is Alg. 8 ("Heuristically parameterise RNS-CKKS
  scheme using expected cost of computation") executed line by line.
* The chain's last entry is the special prime P used only by key-switching; the
  others are the data primes q_0..q_c (reading R1).
* Primes (O2, paper silent): for each bit size in chain order, the largest prime
  p < 2^b with p = 1 mod 2N not already used.
* psi (O3, paper silent): the minimal primitive 2N-th root of unity mod q.
Pinned by tests/test_oracle_params.py (hand traces of Alg. 8 from SPEC.md:248-250,
Miller-Rabin vs trial division / sympy-free brute force, root order checks).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List


def parameterise(c: int, s: int = 40, p: float = 1.5) -> dict:
    """Alg. 8, re-executed literally; also returns m (reading Z4)."""
    if c < 0:
        raise ValueError("cost must be >= 0")
    parms = dict()
    parms["scheme"] = 2                      # PAPER.md:220 "2 is CKKS in MS-SEAL"
    parms["scale"] = pow(2, s)
    m = [s for i in range(c + 2)]
    m[0] = int(m[0] * p)                     # PAPER.md:223 "Mult first special prime"
    m[-1] = int(m[-1] * p)                   # PAPER.md:224 "Mult last special prime"
    b = 27
    while b < sum(m):
        b = b * 2
    parms["poly_modulus_degree"] = int(1024 * (b / 27))
    parms["coeff_mod_bits"] = m              # reading Z4: store the chain too
    return parms


_MR_BASES = (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37)


def is_prime(n: int) -> bool:
    """Deterministic Miller-Rabin for n < 3.3e24 (bases = first 12 primes)."""
    if n < 2:
        return False
    for p in _MR_BASES:
        if n % p == 0:
            return n == p
    d, r = n - 1, 0
    while d % 2 == 0:
        d //= 2
        r += 1
    for a in _MR_BASES:
        x = pow(a, d, n)
        if x == 1 or x == n - 1:
            continue
        for _ in range(r - 1):
            x = x * x % n
            if x == n - 1:
                break
        else:
            return False
    return True


def select_primes(bits: List[int], n: int) -> List[int]:
    """O2: largest unused prime p < 2^b, p = 1 (mod 2N), per entry in chain order."""
    used = set()
    out = []
    two_n = 2 * n
    for b in bits:
        cand = ((1 << b) - 1) // two_n * two_n + 1
        while True:
            if cand < 2:
                raise ValueError("no prime")
            if cand not in used and cand < (1 << b) and is_prime(cand):
                break
            cand -= two_n
        used.add(cand)
        out.append(cand)
    return out


def minimal_psi(q: int, n: int) -> int:
    """O3: the minimal primitive 2N-th root of unity mod q (psi^N = -1)."""
    two_n = 2 * n
    assert (q - 1) % two_n == 0
    x = 2
    while True:
        y = pow(x, (q - 1) // two_n, q)
        if pow(y, n, q) == q - 1:
            break
        x += 1
    # all primitive 2N-th roots are y^t, t odd
    best = q
    yt = y
    y2 = y * y % q
    for _ in range(n):
        if yt < best:
            best = yt
        yt = yt * y2 % q
    return best


@dataclass
class Params:
    """Fixed CKKS parameter set: N, data primes q_0..q_L, special prime P, scale 2^s."""
    n: int
    bits: List[int]
    q: List[int] = field(default_factory=list)      # data primes
    p_special: int = 0
    scale_bits: int = 40
    psi: List[int] = field(default_factory=list)    # per data prime, then P last

    @property
    def L(self) -> int:
        return len(self.q) - 1

    @property
    def moduli(self) -> List[int]:
        return list(self.q) + [self.p_special]

    @property
    def scale(self) -> float:
        return float(2 ** self.scale_bits)


def make_params(n: int, bits: List[int], scale_bits: int = 40) -> Params:
    """bits = full chain incl. the special prime as its last entry (reading R1)."""
    primes = select_primes(bits, n)
    pr = Params(n=n, bits=list(bits), q=primes[:-1], p_special=primes[-1], scale_bits=scale_bits)
    pr.psi = [minimal_psi(m, n) for m in pr.moduli]
    return pr


def params_from_depth(c: int, s: int = 40, p: float = 1.5) -> Params:
    """Alg. 8 then O2/O3: c=2 gives C0 (N=8192, [60,40,40|60]); c=4 gives C1/C3/C4."""
    d = parameterise(c, s, p)
    return make_params(d["poly_modulus_degree"], d["coeff_mod_bits"], s)


def microbench_bits(n_data: int) -> List[int]:
    """C2 chain: [60] + [40]*(L-2) + [60] data limbs, plus one 60-bit P."""
    assert n_data >= 2
    return [60] + [40] * (n_data - 2) + [60] + [60]
