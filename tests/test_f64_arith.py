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


# ---- opt-in switches of arith.cuh / pointwise.cu (DESIGN.md §5 "Measured and rejected"):
# their exactness claims are pinned here with the same exactly rounded emulation.

def _rd(x: Fraction) -> float:
    """Round an exact rational down to binary64 (the device's *_rd operations)."""
    f = float(x)
    if Fraction(f) > x:
        f = math.nextafter(f, -math.inf)
    return f


def shoup_lazy_fq(y: int, w: int, ws: int, q: int) -> int:
    """arith.cuh shoup_lazy_fq: quotient = yh sh (integer) + floor of the cross products
    summed in binary64 with every operation rounded down; returns y w - quotient q."""
    yl, yh, sl, sh = y & 0xFFFFFFFF, y >> 32, ws & 0xFFFFFFFF, ws >> 32
    dsl32 = sl * 2.0 ** -32                       # exact: 32 bits scaled by a power of two
    s = _rd(Fraction(yl) * sh)
    s = _rd(Fraction(yh) * sl + Fraction(s))
    s = _rd(Fraction(yl) * Fraction(dsl32) + Fraction(s))
    t = _rd(Fraction(s) / 2 ** 32 + 2 ** 52)      # 2^52 + floor(s 2^-32)
    return y * w - (yh * sh + int(t) - 2 ** 52) * q


def test_shoup_fq_contract():
    rng = random.Random(5)
    for trial in range(3000):
        bits = rng.choice([33, 45, 59, 60, 61])
        q = rng.getrandbits(bits) | (1 << (bits - 1)) | 1
        w = q - 1 if trial % 7 == 0 else rng.randrange(q)
        ws = (w << 64) // q
        y = rng.choice([(1 << 63) - 1 - rng.getrandbits(8), min(4 * q - 1, (1 << 63) - 1),
                        (rng.getrandbits(31) << 32) | 0xFFFFFFFF, rng.getrandbits(31) << 32, rng.getrandbits(63)])
        r = shoup_lazy_fq(y, w, ws, q)
        assert 0 <= r < 2 * q, (y, w, q, r / q)     # Shoup's [0, 2q) contract for y < 2^63
        assert r % q == (y * w) % q


def test_karatsuba_split_sums_exact():
    """k_cc_mac4 / k_dense_mac3<KARA>: with 22-bit pieces every product is below 2^46, so sums
    of up to 128 products stay below 2^53 (exact in binary64) and S1 = S - S0 - S2 recovers the
    cross terms; the recombination S0 + S1 2^22 + S2 2^44 equals the integer dot product."""
    rng = random.Random(9)
    for terms in (16, 49, 128):
        q = (1 << 44) - 1
        xs = [rng.choice([q - 1, rng.randrange(q)]) for _ in range(terms)]
        ws = [rng.choice([q - 1, rng.randrange(q)]) for _ in range(terms)]
        s0 = s = s2 = 0.0
        for x, w in zip(xs, ws):
            xl, xh, wl, wh = float(x & 0x3FFFFF), float(x >> 22), float(w & 0x3FFFFF), float(w >> 22)
            s0 = fma(xl, wl, s0)
            s = fma(xl + xh, wl + wh, s)
            s2 = fma(xh, wh, s2)
        s1 = s - s0 - s2
        assert max(s0, s, s2) < 2 ** 53 and s1 == int(s1)
        assert int(s0) + int(s1) * 2 ** 22 + int(s2) * 2 ** 44 == sum(x * w for x, w in zip(xs, ws))
        # each sum reduced by f64_reduce is exact and within 0.51 q for any integer |v| < 2^53
        qp = 17592186044399.0   # a 44-bit odd modulus
        for v in (s0, s1, s2):
            rr = f64_reduce(v, qp, 1.0 / qp)
            assert rr == int(rr) and (int(rr) - int(v)) % int(qp) == 0 and abs(rr) <= 0.51 * qp
