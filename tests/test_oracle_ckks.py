"""Pins for oracle/ckks.py: big-integer CRT identities for rescale and key-switch (O11,
O12), keygen error identity (O7), encrypt/decrypt accuracy (O8), homomorphic ops vs
float64, bookkeeping errors (O9)."""
import numpy as np
import pytest

from oracle import ckks, ring
from oracle.params import make_params, params_from_depth
from synth import random_residues


def _ctx(n=64, bits=(60, 40, 40, 40, 60), seed=1):
    return ckks.Context(make_params(n, list(bits))).keygen(seed)


def _crt(residues, qs):
    """Plain CRT with Python ints (independent of oracle.ckks.crt_lift_centered)."""
    Q = 1
    for q in qs:
        Q *= q
    x = 0
    for r, q in zip(residues, qs):
        Mi = Q // q
        x += int(r) * Mi * pow(Mi, -1, q)
    return x % Q, Q


def _centered(x, m):
    x %= m
    return x - m if x > m // 2 else x


def test_rescale_big_int_exact():
    ctx = _ctx()
    lvl = ctx.L
    data = random_residues((2, 2, lvl + 1, ctx.n), ctx.q[: lvl + 1] * 4, seed=3)
    ct = ckks.CtArray(data, lvl, 2.0 ** 80, ctx.key_id)
    out = ctx.rescale(ct)
    qs, ql = ctx.q[:lvl], ctx.q[lvl]
    for c in range(2):
        for k in range(2):
            coef_in = ctx.intt(ct.data[c, k].copy(), list(range(lvl + 1)))
            coef_out = ctx.intt(out.data[c, k].copy(), list(range(lvl)))
            for j in range(ctx.n):
                X, _ = _crt(coef_in[:, j], ctx.q[: lvl + 1])
                want = (X - _centered(X, ql)) // ql
                Qo = 1
                for q in qs:
                    Qo *= q
                got, _ = _crt(coef_out[:, j], qs)
                assert got == want % Qo
    assert out.level == lvl - 1 and out.scale == 2.0 ** 80 / float(ql)


def test_keyswitch_mod_down_big_int_exact():
    ctx = _ctx()
    lvl = 2
    d2 = random_residues((lvl + 1, ctx.n), ctx.q[: lvl + 1], seed=4)
    acc = ctx.keyswitch_acc(d2, lvl)
    out = ctx.mod_down(acc, lvl)
    mods = ctx.q[: lvl + 1] + [ctx.P]
    idx = list(range(lvl + 1)) + [ctx.L + 1]
    Q = 1
    for q in ctx.q[: lvl + 1]:
        Q *= q
    for c in range(2):
        A = ctx.intt(acc[c].copy(), idx)
        O = ctx.intt(out[c].copy(), list(range(lvl + 1)))
        for j in range(ctx.n):
            X, _ = _crt(A[:, j], mods)
            want = ((X - _centered(X, ctx.P)) // ctx.P) % Q
            got, _ = _crt(O[:, j], ctx.q[: lvl + 1])
            assert got == want


def test_keyswitch_acc_is_digit_inner_product():
    """acc over Q*P equals sum_j [d2]_{q_j} * rlk_j exactly (the digit decomposition)."""
    ctx = _ctx()
    lvl = 1
    d2 = random_residues((lvl + 1, ctx.n), ctx.q[: lvl + 1], seed=5)
    acc = ctx.keyswitch_acc(d2, lvl)
    idx = list(range(lvl + 1)) + [ctx.L + 1]
    a = ctx.intt(d2.copy(), list(range(lvl + 1)))
    for c in range(2):
        for ti, t in enumerate(idx):
            m = ctx.moduli[t]
            want = np.zeros(ctx.n, dtype=np.uint64)
            for j in range(lvl + 1):
                x = ctx.ntt(ring.reduce(a[j].copy(), m)[None], [t])[0]
                want = ring.add(want, ring.mul(x, ctx.rlk[j, c, t], m), m)
            assert np.array_equal(acc[c, ti], want)


def test_keygen_error_identity():
    ctx = _ctx(n=256)
    all_idx = list(range(ctx.L + 2))
    for j in range(ctx.L + 1):
        for i in all_idx:
            m = ctx.moduli[i]
            v = ring.add(ctx.rlk[j, 0, i], ring.mul(ctx.rlk[j, 1, i], ctx.s_hat[i], m), m)
            if i == j:
                s2 = ring.mul(ctx.s_hat[i], ctx.s_hat[i], m)
                v = ring.sub(v, ring.mul_scalar(s2, ctx.P % m, m), m)
            e = ctx.intt(v[None].copy(), [i])[0]
            ec = np.array([_centered(int(x), m) for x in e])
            assert np.abs(ec).max() <= 21
    for i in range(ctx.L + 1):
        q = ctx.q[i]
        v = ring.add(ctx.pk[0, i], ring.mul(ctx.pk[1, i], ctx.s_hat[i], q), q)
        e = ctx.intt(v[None].copy(), [i])[0]
        assert [_centered(int(x), q) for x in e] == ctx.pk_e.tolist()


@pytest.fixture(scope="module")
def c0ctx():
    return ckks.Context(params_from_depth(2)).keygen(1)


def test_encrypt_decrypt_accuracy(c0ctx):
    z = np.random.default_rng(0).uniform(0, 1, (3, 4096))
    ct = c0ctx.encrypt(z, enc_seed=2)
    assert ct.data.shape == (3, 2, 3, 8192)
    back = c0ctx.decrypt(ct, 4096)
    assert np.max(np.abs(back - z)) < 1e-6


def test_homomorphic_linear_ops(c0ctx):
    rng = np.random.default_rng(1)
    z1, z2 = rng.uniform(-1, 1, (2, 2, 4096))
    a = c0ctx.encrypt(z1, 2, obj0=0)
    b = c0ctx.encrypt(z2, 2, obj0=10)
    s = c0ctx.decrypt(c0ctx.add(a, b), 4096)
    assert np.max(np.abs(s - (z1 + z2))) < 1e-6
    w = [0.3, -1.7]
    m = c0ctx.rescale(c0ctx.mul_scalar(a, w, float(c0ctx.q[2])))
    assert np.max(np.abs(c0ctx.decrypt(m, 4096) - z1 * np.array(w)[:, None])) < 1e-6
    p = c0ctx.add_scalar(a, [0.5, -2.0])
    assert np.max(np.abs(c0ctx.decrypt(p, 4096) - (z1 + np.array([0.5, -2.0])[:, None]))) < 1e-6


def test_mul_relin_rescale(c0ctx):
    rng = np.random.default_rng(2)
    z1, z2 = rng.uniform(-1, 1, (2, 1, 4096))
    a = c0ctx.encrypt(z1, 2, obj0=0)
    b = c0ctx.encrypt(z2, 2, obj0=1)
    d, lvl, sc = c0ctx.tensor(a, b)
    # decrypt the 3-component ciphertext with (1, s, s^2) before relinearising
    q0 = c0ctx.q[0]
    m3 = ring.add(ring.add(d[0, 0, 0], ring.mul(d[0, 1, 0], c0ctx.s_hat[0], q0), q0),
                  ring.mul(d[0, 2, 0], ring.mul(c0ctx.s_hat[0], c0ctx.s_hat[0], q0), q0), q0)
    r = c0ctx.mul_relin(a, b)
    m2 = ring.add(r.data[0, 0, 0], ring.mul(r.data[0, 1, 0], c0ctx.s_hat[0], q0), q0)
    diff = ring.sub(c0ctx.intt(m3[None].copy(), [0])[0], c0ctx.intt(m2[None].copy(), [0])[0], q0)
    dc = np.array([_centered(int(x), q0) for x in diff])
    # relinearisation noise bound: (l+1) N 21 max q / P + N, in integer units
    bound = (lvl + 1) * c0ctx.n * 21 * max(c0ctx.q) / c0ctx.P + c0ctx.n
    assert np.abs(dc).max() <= bound
    out = c0ctx.decrypt(c0ctx.rescale(r), 4096)
    assert np.max(np.abs(out - z1 * z2)) < 1e-5


def test_bookkeeping_errors(c0ctx):
    z = np.zeros((1, 16))
    a = c0ctx.encrypt(z, 2)
    x = a
    for _ in range(c0ctx.L):            # depth sufficiency: exactly L rescales
        x = c0ctx.rescale(c0ctx.mul_scalar(x, [1.0], float(c0ctx.q[x.level])))
    with pytest.raises(ckks.LevelError):
        c0ctx.rescale(x)
    other = ckks.Context(params_from_depth(2)).keygen(7)
    with pytest.raises(ckks.KeyMismatch):
        other.decrypt(a, 16)
    b = c0ctx.mul_scalar(a, [1.0], 3.0)
    with pytest.raises(ckks.ScaleError):
        c0ctx.add(a, b)
    with pytest.raises(ckks.CapacityError):
        c0ctx.encrypt(np.zeros((1, 4097)), 2)
    with pytest.raises(ckks.ShapeMismatch):
        c0ctx.add(a, c0ctx.encrypt(np.zeros((2, 16)), 2))
    # auto mod-drop: adding a lower-level operand drops the higher one
    lo = c0ctx.rescale(c0ctx.mul_scalar(a, [1.0], float(c0ctx.q[2])))
    s = c0ctx.add(lo, a)
    assert s.level == 1


def test_encrypt_sk_error_identity(c0ctx):
    """Secret-key encryption (DESIGN reading Z16): c0 + c1 s = m + e exactly, with e the
    TAG_SK_E CBD sample and the decryption pinned above; c1 is the seeded uniform draw."""
    from oracle import sampling as smp
    rng = np.random.default_rng(5)
    polys = rng.integers(-2 ** 40, 2 ** 40, (2, c0ctx.n))
    ct = c0ctx.encrypt_poly_sk(polys, enc_seed=9, obj0=4, scale=2.0 ** 40)
    assert ct.data.shape == (2, 2, c0ctx.L + 1, c0ctx.n)
    dec = c0ctx.decrypt_poly(ct)
    k_e = ckks.sk_error_key(c0ctx.sk_seed, 9)
    for c in range(2):
        e = smp.cbd(c0ctx.n, k_e, 4 + c, smp.TAG_SK_E)
        assert dec[c] == [int(m) + int(x) for m, x in zip(polys[c], e)]
        # the error is not the stream of the public wire seed (anyone holding c0
        # and enc_seed could otherwise strip the noise)
        e_pub = smp.cbd(c0ctx.n, 9, 4 + c, smp.TAG_SK_E)
        assert not np.array_equal(e, e_pub)
        for i in range(c0ctx.L + 1):
            assert np.array_equal(ct.data[c, 1, i], smp.uniform(c0ctx.n, 9, 4 + c, i, smp.TAG_SK_A, c0ctx.q[i]))


def test_encrypt_sk_homomorphic(c0ctx):
    """A secret-key ciphertext computes with public-key ones under the same key."""
    rng = np.random.default_rng(6)
    z1, z2 = rng.uniform(-1, 1, (2, 1, 4096))
    sc = c0ctx.p.scale
    a = c0ctx.encrypt_poly_sk(np.stack([c0ctx.encode(z1[0], sc)]), 3, 0, sc)
    b = c0ctx.encrypt(z2, 2, obj0=1)
    m = c0ctx.rescale(c0ctx.mul_relin(a, b))
    assert np.max(np.abs(c0ctx.decrypt(m, 4096) - z1 * z2)) < 1e-5
    assert np.max(np.abs(c0ctx.decrypt(a, 4096) - z1)) < 1e-6


def _negacyclic_int(a, b):
    """Exact negacyclic product of two small-integer polynomials (schoolbook via a linear
    convolution, then X^N = -1 folding)."""
    n = len(a)
    full = np.convolve(np.asarray(a, dtype=np.int64), np.asarray(b, dtype=np.int64))
    out = full[:n].copy()
    out[: n - 1] -= full[n:]
    return out


def test_encrypt_pk_error_identity(c0ctx):
    """O8 public-key encryption pinned exactly: with pk = (b, a),
    b = -a s + e_pk, the ciphertext (v b + e0 + m, v a + e1) decrypts to
    c0 + c1 s = m + v e_pk + e0 + e1 s, a negacyclic identity over the integers that is
    checked coefficient by coefficient with the sampled v (ternary), e0, e1 (CBD), the
    secret s and the key's error e_pk.  Dropping e0 or e1, drawing v from the CBD, or a
    wrong sign anywhere breaks it."""
    from oracle import sampling as smp
    rng = np.random.default_rng(15)
    polys = rng.integers(-2 ** 40, 2 ** 40, (2, c0ctx.n))
    ct = c0ctx.encrypt_poly(polys, enc_seed=7, obj0=3, scale=2.0 ** 40)
    dec = c0ctx.decrypt_poly(ct)
    s = c0ctx.s_coef
    for c in range(2):
        v = smp.ternary(c0ctx.n, 7, 3 + c, smp.TAG_ENC_V)
        e0 = smp.cbd(c0ctx.n, 7, 3 + c, smp.TAG_ENC_E0)
        e1 = smp.cbd(c0ctx.n, 7, 3 + c, smp.TAG_ENC_E1)
        assert set(np.unique(v)) <= {-1, 0, 1}
        noise = _negacyclic_int(v, c0ctx.pk_e) + e0 + _negacyclic_int(e1, s)
        assert dec[c] == [int(m) + int(x) for m, x in zip(polys[c], noise)]


def test_key_identifier_is_not_the_seed(c0ctx):
    """the public key_id is a one-way function of the secret seed."""
    import hashlib
    seed = c0ctx.sk_seed
    assert c0ctx.key_id != seed
    d = hashlib.sha256(b"edl-key\0" + seed.to_bytes(8, "little")).digest()
    assert c0ctx.key_id == int.from_bytes(d[:8], "little")
