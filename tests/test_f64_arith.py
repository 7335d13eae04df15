"""Host-side check of the FP64-pipe modular arithmetic's error analysis (DESIGN.md §5,
`csrc/arith.cuh` f64_mulc / f64_reduce), independent of the GPU: the same operation
sequence evaluated with exactly rounded binary64 arithmetic (FMA emulated with Python's
exact rationals, round-to-nearest-even) must give a result congruent to b w mod q and
inside the claimed range, for moduli up to the path's threshold q < 2^44 and operands up
to |b| < 2^50.  (Test infrastructure; no oracle code involved.)"""
import math
import random
from fractions import Fraction

import pytest

RND = 6755399441055744.0      # 1.5 * 2^52


def fma(a: float, b: float, c: float) -> float:
    """Correctly rounded a*b + c (float(Fraction) rounds to nearest, ties to even)."""
    return float(Fraction(a) * Fraction(b) + Fraction(c))


def rd_div(w: int, q: int) -> float:
    """RD(w / q) as binary64."""
    x = float(Fraction(w, q))
    if Fraction(x) > Fraction(w, q):
        x = math.nextafter(x, -math.inf)
    return x


def f64_mulc(b: float, w: float, wq: float, q: float) -> float:
    hi = b * w
    lo = fma(b, w, -hi)
    qt = fma(b, wq, RND) - RND
    return fma(-qt, q, hi) + lo


def f64_reduce(v: float, q: float, qinv: float) -> float:
    qt = fma(v, qinv, RND) - RND
    return fma(-qt, q, v)


def _cases(seed, n=400):
    rng = random.Random(seed)
    for _ in range(n):
        bits = rng.choice([20, 30, 36, 40, 41, 43, 44])
        q = rng.randrange(2 ** (bits - 1), 2 ** bits) | 1
        w = rng.choice([0, 1, q - 1, rng.randrange(q)])
        bmax = 2 ** 50 - 1
        b = rng.choice([bmax, -bmax, 15 * q, -15 * q, rng.randrange(-bmax, bmax + 1)])
        yield q, w, b


@pytest.mark.parametrize("seed", [1, 2])
def test_f64_mulc_exact_and_bounded(seed):
    for q, w, b in _cases(seed):
        t = f64_mulc(float(b), float(w), rd_div(w, q), float(q))
        assert t == int(t), (q, w, b)
        assert (int(t) - b * w) % q == 0, (q, w, b)
        assert abs(t) <= 0.625 * q, (q, w, b, t / q)


@pytest.mark.parametrize("seed", [3, 4])
def test_f64_reduce_exact_and_bounded(seed):
    for q, _, b in _cases(seed):
        r = f64_reduce(float(b), float(q), 1.0 / q)
        assert r == int(r) and (int(r) - b) % q == 0
        assert abs(r) <= 0.51 * q


def test_forward_growth_bound():
    """Forward transform: inputs < 4q, each of up to 16 stages adds at most 0.625 q, so every
    intermediate stays below 15 q < 2^50 for q < 2^44 (the f64_mulc operand bound)."""
    q = 2 ** 44 - 1
    assert 4 * q + 16 * 0.625 * q < 15 * q < 2 ** 50
    # inverse: a pass of <= 5 stages starts below 2q; its last-stage differences reach 2q 2^5
    assert 2 * q * 2 ** 5 < 2 ** 50
