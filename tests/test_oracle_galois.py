"""Pins for the oracle's Galois rotations, plaintext-vector products and kernel
masquerading (NEXT f1): group identities of the automorphism,
decrypt(rotate(encrypt(z), r)) == z rotated by r, masked cross-correlation == the float64
cross-correlation at every window anchor."""
import numpy as np
import pytest

from oracle import ckks, galois, networks, ring
from oracle.params import make_params


@pytest.fixture(scope="module")
def small():
    ctx = ckks.Context(make_params(1024, [60, 40, 40, 40, 40, 60])).keygen(1)
    return ctx


def test_automorphism_group_identities(small):
    ctx = small
    n, q = ctx.n, ctx.q[1]
    a = np.random.default_rng(0).integers(0, q, n, dtype=np.uint64)
    assert np.array_equal(galois.automorphism_coeff(a, 1, q), a)
    for g, h in ((5, 25), (3, 7), (5, 2 * n - 1)):
        lhs = galois.automorphism_coeff(galois.automorphism_coeff(a, h, q), g, q)
        assert np.array_equal(lhs, galois.automorphism_coeff(a, (g * h) % (2 * n), q))
    # X -> X^(2N-1) = -X^(N-1) on the monomial X
    x = np.zeros(n, dtype=np.uint64)
    x[1] = 1
    y = galois.automorphism_coeff(x, 2 * n - 1, q)
    assert int(y[n - 1]) == q - 1 and int(y.sum()) == q - 1
    assert galois.galois_element(0, n) == 1 and galois.galois_element(1, n) == 5
    assert galois.galois_element(-1, n) * 5 % (2 * n) == 1


def test_automorphism_ntt_matches_coefficients(small):
    ctx = small
    idx = [0, 1]
    a = np.random.default_rng(1).integers(0, ctx.q[1], (2, ctx.n), dtype=np.uint64)
    a[0] %= np.uint64(ctx.q[0])
    a_hat = ctx.ntt(a.copy(), idx)
    got = ctx.intt(galois.automorphism_ntt(ctx, a_hat, 25, idx), idx)
    for r, i in enumerate(idx):
        assert np.array_equal(got[r], galois.automorphism_coeff(a[r], 25, ctx.q[i]))


@pytest.mark.parametrize("r", [1, 3, -2])
def test_rotation_decrypts_to_rotated_slots(small, r):
    ctx = small
    z = np.random.default_rng(2).uniform(-1, 1, (2, ctx.n // 2))
    x = ctx.encrypt(z, 2)
    gk = {galois.galois_element(r, ctx.n): galois.galois_keygen(ctx, 7, galois.galois_element(r, ctx.n))}
    y = galois.rotate(ctx, x, r, gk)
    assert y.level == x.level and y.scale == x.scale
    assert np.max(np.abs(ctx.decrypt(y, ctx.n // 2) - np.roll(z, -r, axis=1))) < 1e-5


def test_hoisted_rotations_decrypt_to_rotated_slots(small):
    """rotate_hoisted (one modulus raise shared by several rotations) decrypts to the rotated
    slots, and its c0/c1 differ from the plain rotation's only within the key-switch noise."""
    ctx = small
    z = np.random.default_rng(4).uniform(-1, 1, (2, ctx.n // 2))
    x = ctx.encrypt(z, 2)
    rs = [1, -2, 5]
    gk = {galois.galois_element(r, ctx.n): galois.galois_keygen(ctx, 7, galois.galois_element(r, ctx.n)) for r in rs}
    ys = galois.rotate_hoisted(ctx, x, rs, gk)
    for r, y in zip(rs, ys):
        assert y.level == x.level and y.scale == x.scale
        assert np.max(np.abs(ctx.decrypt(y, ctx.n // 2) - np.roll(z, -r, axis=1))) < 1e-5
        y0 = galois.rotate(ctx, x, r, gk)
        d = np.abs(ctx.decrypt(y, ctx.n // 2) - ctx.decrypt(y0, ctx.n // 2))
        assert d.max() < 1e-6 and not np.array_equal(y.data, y0.data)


def test_plain_vector_product(small):
    ctx = small
    rng = np.random.default_rng(3)
    z, w = rng.uniform(-1, 1, (2, 512)), rng.uniform(-1, 1, 512)
    x = ctx.encrypt(z, 2)
    l = x.level
    pt = galois.encode_plain(ctx, w, float(ctx.q[l]), l)
    y = ctx.rescale(galois.mul_plain(ctx, x, np.broadcast_to(pt, (2,) + pt.shape), float(ctx.q[l])))
    assert np.max(np.abs(ctx.decrypt(y, 512) - z * w)) < 1e-5


def test_masked_cc_matches_float64(small):
    """Kernel masquerading + rotation sums on an 8x8 image, 2 filters 4x4 stride 4."""
    ctx = small
    rng = np.random.default_rng(4)
    imgs = rng.integers(0, 256, (2, 8, 8)) / 255.0
    K, kb = rng.normal(0, 0.1, (2, 4, 4)), rng.normal(0, 0.1, 2)
    slots = np.zeros((2, ctx.n // 2))
    slots[:, :64] = imgs.reshape(2, 64)
    x = ctx.encrypt(slots, 2)
    rots = galois.window_rotations(4, 4, 8)
    assert rots == [1, 2, 8, 16]
    gk = {galois.galois_element(r, ctx.n): galois.galois_keygen(ctx, 7, galois.galois_element(r, ctx.n)) for r in rots}
    y = galois.masked_cc(ctx, x, K, 8, 8, 4, kb, gk)
    assert y.count == 4 and y.level == x.level - 1
    dec = ctx.decrypt(y, 64).reshape(2, 2, 64)                     # [image][filter][slot]
    want = networks.cc_float64(imgs, K, kb)                         # [image][filter*windows]
    for b in range(2):
        for f in range(2):
            for rr in range(2):
                for cc in range(2):
                    got = dec[b, f, (rr * 4) * 8 + cc * 4]
                    assert abs(got - want[b, f * 4 + rr * 2 + cc]) < 1e-4


# ------------------------------------------------------------------ packed paper-layout CNN
F1_H, F1_W, F1_K, F1_F, F1_O = 16, 16, 4, 2, 3


def _f1_small_net():
    rw = np.random.default_rng(41)
    K = rw.normal(0.0, 0.1, (F1_F, F1_K, F1_K))
    kb = rw.normal(0.0, 0.1, F1_F)
    A = (F1_H // F1_K) * (F1_W // F1_K)
    Wt = rw.normal(0.0, 0.1, (F1_O, F1_F * A))
    b = rw.normal(0.0, 0.1, F1_O)
    imgs = np.random.default_rng(42).integers(0, 256, (2, F1_H, F1_W)) / 255.0
    return K, kb, Wt, b, imgs


def f1_rotations(n_slots):
    """Tap rotations of the hoisted CC + replication and block-sum rotations of the packed dense."""
    taps = [u * F1_W + v for u in range(F1_K) for v in range(F1_K) if u or v]
    blk = 1
    while blk < F1_H * F1_W:
        blk *= 2
    reps, s = [], blk
    while s < n_slots:
        reps.append(n_slots - s)
        s *= 2
    sums, s = [], 1
    while s < blk:
        sums.append(s)
        s *= 2
    return sorted(set(taps + reps + sums))


@pytest.fixture(scope="module")
def f1_small_oracle(small):
    ctx = small
    gk = {galois.galois_element(r, ctx.n): galois.galois_keygen(ctx, 7, galois.galois_element(r, ctx.n))
          for r in f1_rotations(ctx.n // 2)}
    K, kb, Wt, b, imgs = _f1_small_net()
    x = ctx.encrypt(imgs.reshape(2, -1), 2)
    out = galois.masked_cnn_packed(ctx, x, K, kb, Wt, b, F1_H, F1_W, F1_K, networks.SIGMA_A, gk, ctx.encode)
    return out, gk


def test_masked_cnn_packed_vs_float64(small, f1_small_oracle):
    """the oracle twin of the GPU's hoisted masked CC + class-packed dense
    (with the sigma(kb) compensation) decrypts to the float64 network within 1e-3
    (N = 2^10, 16x16 images, 2 filters 4x4 stride 4, dense 32 -> 3; 2 product ciphertexts
    per image because 2 classes fit in the 512 slots)."""
    ctx = small
    out, _ = f1_small_oracle
    K, kb, Wt, b, imgs = _f1_small_net()
    assert out.count == 2 * 2 and out.level == 0
    got = galois.packed_logits(ctx, out, F1_O, F1_H * F1_W)
    ref = networks.c1_float64(imgs, K, kb, Wt, b)
    assert ref.shape == got.shape == (2, F1_O)
    assert np.max(np.abs(got - ref)) < 1e-3
