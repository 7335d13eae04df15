"""GPU parity: the CUDA path (through the C-ABI) against the oracle, element by element.

Integer work is compared bit-exactly on every residue (the north_star's bar); decrypted
values within 1e-3 of float64.  Sizes span several tiles and ragged counts.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import ckks as ock, layers as olay, networks as onet, ring as oring  # noqa: E402
from oracle.params import make_params, params_from_depth  # noqa: E402
from synth import random_residues, c0_inputs, random_slots  # noqa: E402


@pytest.fixture(scope="module")
def edl():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2110_13638_b200 import edl as E
    return E


def _pair(E, depth=None, logn=None, bits=None, seed=1):
    if depth is not None:
        pp = E.params_from_depth(depth)
        po = params_from_depth(depth)
    else:
        pp = E.params_from_bits(logn, bits)
        po = make_params(1 << logn, list(bits))
    assert pp.qs == po.q and pp.p_special == po.p_special and pp.psis == po.psi
    g = E.Context(pp).keygen(seed)
    o = ock.Context(po).keygen(seed)
    return g, o


@pytest.fixture(scope="module")
def c0pair(edl):
    return _pair(edl, depth=2)


@pytest.fixture(scope="module")
def c1pair(edl):
    return _pair(edl, depth=4)


def _rand_ct(o, cnt, lvl, seed):
    mods = o.q[: lvl + 1] * (cnt * 2)
    return random_residues((cnt, 2, lvl + 1, o.n), mods, seed=seed)


def _to_gpu(g, data, lvl, scale, key):
    return g.from_numpy(data, lvl, scale, key)


# ---------------------------------------------------------------- NTT
@pytest.mark.parametrize("logn", [10, 11, 12, 13, 14, 15, 16])
def test_ntt_bit_exact(edl, logn):
    bits = [60, 40, 40, 60] if logn < 14 else [60, 40, 40, 40, 40, 60]
    pp = edl.params_from_bits(logn, bits)
    g = edl.Context(pp)
    po = make_params(1 << logn, bits)
    lvl = len(bits) - 2
    n_polys = 3
    mods = po.q[: lvl + 1] * n_polys
    psis = po.psi[: lvl + 1] * n_polys
    a = random_residues((n_polys, lvl + 1, 1 << logn), mods, seed=logn)
    t = torch.from_numpy(a.view(np.int64).reshape(-1).copy()).cuda()
    g.ntt_(t, n_polys, lvl, inverse=False)
    got = t.cpu().numpy().view(np.uint64).reshape(a.shape)
    want = oring.ntt_fwd(a, mods, psis)
    assert np.array_equal(got, want)
    g.ntt_(t, n_polys, lvl, inverse=True)
    back = t.cpu().numpy().view(np.uint64).reshape(a.shape)
    assert np.array_equal(back, a)
    # inverse of arbitrary residues too
    t2 = torch.from_numpy(a.view(np.int64).reshape(-1).copy()).cuda()
    g.ntt_(t2, n_polys, lvl, inverse=True)
    assert np.array_equal(t2.cpu().numpy().view(np.uint64).reshape(a.shape), oring.ntt_inv(a, mods, psis))


def test_ntt_large_batch_sampled(edl):
    """C2-sized batches (several work items per persistent cluster, ragged tail): sampled
    polynomials of a 301-poly batch at N = 2^14 against the oracle, forward and inverse."""
    bits = [60, 40, 40, 40, 40, 60]
    g = edl.Context(edl.params_from_bits(14, bits))
    po = make_params(1 << 14, bits)
    lvl, n_polys = 4, 301
    a = random_residues((n_polys, lvl + 1, 1 << 14), po.q[: lvl + 1] * n_polys, seed=77)
    t = torch.from_numpy(a.view(np.int64).reshape(-1).copy()).cuda()
    g.ntt_(t, n_polys, lvl, inverse=False)
    got = t.cpu().numpy().view(np.uint64).reshape(a.shape)
    for k in (0, 1, 150, 299, 300):
        assert np.array_equal(got[k], oring.ntt_fwd(a[k], po.q[: lvl + 1], po.psi[: lvl + 1])), k
    g.ntt_(t, n_polys, lvl, inverse=True)
    assert np.array_equal(t.cpu().numpy().view(np.uint64).reshape(a.shape), a)


@pytest.mark.parametrize("logn", [12, 14, 16])
def test_ntt_prime_classes(edl, logn):
    """Every butterfly path of the NTT core against the oracle: q < 2^44 (FP64-pipe
    butterflies: 30- and 44-bit primes), 2^44 <= q < 2^46 (Shoup butterflies, FP64-quotient
    constants: 45 bits), and Shoup with integer constants (50, 60 bits); one polynomial of
    all-(q-1) residues drives the unreduced FP64 intermediates to their largest values."""
    bits = [60, 30, 44, 45, 50, 60]
    pp = edl.params_from_bits(logn, bits)
    g = edl.Context(pp)
    po = make_params(1 << logn, bits)
    lvl = len(bits) - 2
    n_polys = 3
    mods = po.q[: lvl + 1] * n_polys
    psis = po.psi[: lvl + 1] * n_polys
    a = random_residues((n_polys, lvl + 1, 1 << logn), mods, seed=logn + 100)
    for i in range(lvl + 1):
        a[0, i, :] = np.uint64(po.q[i] - 1)
    for inverse in (False, True):
        t = torch.from_numpy(a.view(np.int64).reshape(-1).copy()).cuda()
        g.ntt_(t, n_polys, lvl, inverse=inverse)
        got = t.cpu().numpy().view(np.uint64).reshape(a.shape)
        want = (oring.ntt_inv if inverse else oring.ntt_fwd)(a, mods, psis)
        assert np.array_equal(got, want), ("inverse" if inverse else "forward")


def test_ntt_special_prime_limb(edl):
    pp = edl.params_from_depth(2)
    g = edl.Context(pp)
    po = params_from_depth(2)
    n = po.n
    a = random_residues((2, 4, n), po.moduli * 2, seed=9)
    t = torch.from_numpy(a.view(np.int64).reshape(-1).copy()).cuda()
    g.ntt_(t, 2, 3)   # level L+1 = includes P as limb 3
    assert np.array_equal(t.cpu().numpy().view(np.uint64).reshape(a.shape), oring.ntt_fwd(a, po.moduli * 2, po.psi * 2))


# ---------------------------------------------------------------- Philox / keys / encryption
def test_philox_words(edl, c0pair):
    from oracle import sampling
    g, _ = c0pair
    rng = np.random.default_rng(0)
    ctr = rng.integers(0, 2 ** 32, (257, 4), dtype=np.uint64).astype(np.uint32)
    for seed in (0, 1, 0xDEADBEEFCAFEF00D):
        got = g.philox(seed, ctr)
        want = np.stack([sampling.philox4x32_10(c, (seed & 0xFFFFFFFF, seed >> 32)) for c in ctr])
        assert np.array_equal(got, want)


@pytest.mark.parametrize("which", ["c0", "c1"])
def test_keygen_bit_exact(which, c0pair, c1pair):
    g, o = c0pair if which == "c0" else c1pair
    # public key identifier: SHA-256 of the seed on both sides (host C++ vs hashlib), never the seed
    assert g.key_id == o.key_id != o.sk_seed
    assert np.array_equal(g.export_key(0), o.s_hat)
    assert np.array_equal(g.export_key(1), o.pk)
    assert np.array_equal(g.export_key(2), o.rlk)


@pytest.mark.parametrize("level", [None, 1])
def test_encrypt_bit_exact(c1pair, level):
    g, o = c1pair
    z = random_slots(5, 8192, seed=3)
    polys = np.stack([o.encode(v) for v in z])            # same integer polys on both sides (Z1)
    want = o.encrypt_poly(polys, enc_seed=2, obj0=7, scale=o.p.scale, level=level)
    got = g.encrypt_poly(polys, scale=o.p.scale, enc_seed=2, obj0=7, level=level)
    assert got.level == want.level and got.count == 5
    assert np.array_equal(got.numpy(g.n), want.data)


def test_encode_contract(c1pair):
    """Z1: host FFT encode vs oracle encode: |dm| <= 1 and <= 1% of coefficients differ."""
    g, o = c1pair
    z = random_slots(3, 8192, seed=5)
    got = g.encode(z)
    want = np.stack([o.encode(v) for v in z])
    d = np.abs(got - want)
    assert d.max() <= 1 and (d > 0).mean() <= 0.01


def test_decrypt_matches_oracle(c0pair):
    g, o = c0pair
    z = random_slots(4, 4096, seed=6, lo=-1, hi=1)
    polys = np.stack([o.encode(v) for v in z])
    ct_g = g.encrypt_poly(polys, scale=o.p.scale, enc_seed=2)
    ct_o = o.encrypt_poly(polys, 2, 0, o.p.scale)
    dp = g.decrypt_poly(ct_g)
    want = np.array(o.decrypt_poly(ct_o), dtype=object)
    assert [[int(v) for v in row] for row in dp] == [[int(v) for v in row] for row in want]
    assert np.max(np.abs(g.decrypt(ct_g, 4096) - z)) < 1e-6


# ---------------------------------------------------------------- ciphertext ops
@pytest.mark.parametrize("cnt", [1, 3, 7])
def test_ops_bit_exact(c1pair, cnt):
    g, o = c1pair
    L = o.L
    sc = o.p.scale
    A = ock.CtArray(_rand_ct(o, cnt, L, 11 + cnt), L, sc, o.key_id)
    B = ock.CtArray(_rand_ct(o, cnt, L, 12 + cnt), L, sc, o.key_id)
    ga, gb = _to_gpu(g, A.data, L, sc, o.key_id), _to_gpu(g, B.data, L, sc, o.key_id)
    assert np.array_equal(g.add(ga, gb).numpy(g.n), o.add(A, B).data)
    w = np.linspace(-1.5, 2.0, cnt)
    assert np.array_equal(g.pt_mul(ga, w, 2.0 ** 30).numpy(g.n), o.mul_scalar(A, w, 2.0 ** 30).data)
    assert np.array_equal(g.pt_add(ga, w).numpy(g.n), o.add_scalar(A, w).data)
    r_g, r_o = g.rescale(ga), o.rescale(A)
    assert r_g.level == r_o.level and r_g.scale == r_o.scale
    assert np.array_equal(r_g.numpy(g.n), r_o.data)
    assert np.array_equal(g.mod_drop(ga, 2).numpy(g.n), o.mod_drop(A, 2).data)
    # add with auto mod-drop of the higher operand (operands at matching scales)
    B2 = ock.CtArray(B.data, L, r_o.scale, o.key_id)
    gb2 = _to_gpu(g, B.data, L, r_o.scale, o.key_id)
    s_g, s_o = g.add(r_g, gb2), o.add(r_o, B2)
    assert s_g.level == s_o.level == L - 1
    assert np.array_equal(s_g.numpy(g.n), s_o.data)


@pytest.mark.parametrize("lvl", [1, 2, 3, 4])
def test_mul_relin_bit_exact(c1pair, lvl):
    g, o = c1pair
    cnt = 2
    A = ock.CtArray(_rand_ct(o, cnt, lvl, 21 + lvl), lvl, 2.0 ** 40, o.key_id)
    B = ock.CtArray(_rand_ct(o, cnt, lvl, 31 + lvl), lvl, 2.0 ** 40, o.key_id)
    got = g.mul_relin(_to_gpu(g, A.data, lvl, A.scale, o.key_id), _to_gpu(g, B.data, lvl, B.scale, o.key_id))
    want = o.mul_relin(A, B)
    assert got.scale == want.scale
    assert np.array_equal(got.numpy(g.n), want.data)


def test_fused_keyswitch_bit_exact(edl, monkeypatch):
    """The fused target-major key switch (k_relin_ks, EDL_KS_FUSED=1) against the oracle:
    mul_relin at every level of the C1 chain (16 ciphertexts: both stream halves), and the
    sigma_a layer (two key switches, one with the fused output assembly)."""
    monkeypatch.setenv("EDL_KS_FUSED", "1")
    g, o = _pair(edl, depth=4)
    for lvl in (1, 2, 3, 4):
        A = ock.CtArray(_rand_ct(o, 16, lvl, 121 + lvl), lvl, 2.0 ** 40, o.key_id)
        B = ock.CtArray(_rand_ct(o, 16, lvl, 131 + lvl), lvl, 2.0 ** 40, o.key_id)
        got = g.mul_relin(_to_gpu(g, A.data, lvl, A.scale, o.key_id), _to_gpu(g, B.data, lvl, B.scale, o.key_id))
        assert np.array_equal(got.numpy(g.n), o.mul_relin(A, B).data), lvl
    X = ock.CtArray(_rand_ct(o, 3, 3, 141), 3, 2.0 ** 40, o.key_id)
    got = g.poly_activation(_to_gpu(g, X.data, 3, X.scale, o.key_id), [0.5, 0.197, 0.0, -0.004])
    want = olay.poly_activation(o, X, [0.5, 0.197, 0.0, -0.004])
    assert np.array_equal(got.numpy(g.n), want.data)


@pytest.mark.parametrize("logn", [15, 16])
def test_large_n_keys_relin_rescale(edl, logn):
    """C2's large rings (one limb per thread-block cluster of N/2^13 CTAs): keygen, encryption,
    tensor + key-switch (with and without the fused rescale) and rescale, bit-exact."""
    bits = [60, 40, 40, 60]
    g, o = _pair(edl, logn=logn, bits=bits, seed=5)
    assert np.array_equal(g.export_key(0), o.s_hat)
    assert np.array_equal(g.export_key(1), o.pk)
    assert np.array_equal(g.export_key(2), o.rlk)
    polys = np.random.default_rng(logn).integers(-2 ** 30, 2 ** 30, (2, 1 << logn))
    xg = g.encrypt_poly(polys, scale=2.0 ** 40, enc_seed=7)
    xo = o.encrypt_poly(polys, enc_seed=7, obj0=0, scale=2.0 ** 40)
    assert np.array_equal(xg.numpy(g.n), xo.data)
    lvl = 2
    A = ock.CtArray(_rand_ct(o, 2, lvl, 51), lvl, 2.0 ** 40, o.key_id)
    B = ock.CtArray(_rand_ct(o, 2, lvl, 52), lvl, 2.0 ** 40, o.key_id)
    ga, gb = _to_gpu(g, A.data, lvl, A.scale, o.key_id), _to_gpu(g, B.data, lvl, B.scale, o.key_id)
    m_g, m_o = g.mul_relin(ga, gb), o.mul_relin(A, B)
    assert np.array_equal(m_g.numpy(g.n), m_o.data)
    assert np.array_equal(g.rescale(m_g).numpy(g.n), o.rescale(m_o).data)
    sq_g = g.poly_activation(ga, (0.0, 0.0, 1.0))
    sq_o = olay.poly_activation(o, A, (0.0, 0.0, 1.0))
    assert np.array_equal(sq_g.numpy(g.n), sq_o.data)


def test_mul_relin_c2_chain_batch(edl):
    """C2's L=3 chain (60, 40, 60 | 60: the last data limb on the integer path) with a batch
    of 64 ciphertexts: tensor + key-switch and the following rescale on the GPU, the last
    two ciphertexts (whose successors lie past the array end) checked against the oracle."""
    g, o = _pair(edl, logn=13, bits=[60, 40, 60, 60], seed=7)
    lvl, cnt = 2, 64
    A = ock.CtArray(_rand_ct(o, cnt, lvl, 61), lvl, 2.0 ** 40, o.key_id)
    B = ock.CtArray(_rand_ct(o, cnt, lvl, 62), lvl, 2.0 ** 40, o.key_id)
    m_g = g.mul_relin(_to_gpu(g, A.data, lvl, A.scale, o.key_id), _to_gpu(g, B.data, lvl, B.scale, o.key_id))
    r_g = g.rescale(m_g)
    tail = slice(cnt - 2, cnt)
    At = ock.CtArray(A.data[tail], lvl, A.scale, o.key_id)
    Bt = ock.CtArray(B.data[tail], lvl, B.scale, o.key_id)
    m_o = o.mul_relin(At, Bt)
    assert np.array_equal(m_g.numpy(g.n)[tail], m_o.data)
    assert np.array_equal(r_g.numpy(g.n)[tail], o.rescale(m_o).data)


@pytest.mark.parametrize("which", ["c0", "c1"])
def test_encrypt_sk_and_seeded_wire(which, c0pair, c1pair):
    """Secret-key encryption (reading Z16) bit-exact against the oracle; the seeded wire
    format (c0 packed, c1 regenerated from the seed on the device) reproduces the arrays."""
    g, o = c0pair if which == "c0" else c1pair
    rng = np.random.default_rng(17)
    polys = rng.integers(-2 ** 40, 2 ** 40, (5, o.n))
    xg = g.encrypt_poly_sk(polys, scale=2.0 ** 40, enc_seed=21, obj0=3)
    xo = o.encrypt_poly_sk(polys, enc_seed=21, obj0=3, scale=2.0 ** 40)
    assert np.array_equal(xg.numpy(g.n), xo.data)
    wire = g.pack_c0(xg)
    assert wire.numel() * 8 == g.seeded_bytes(5, g.L) == g.packed_bytes(5, g.L) // 2
    back = g.unpack_seeded(wire, 5, g.L, xg.scale, xg.key_id, enc_seed=21, obj0=3)
    assert np.array_equal(back.numpy(g.n), xo.data)
    assert np.allclose(g.decrypt(back, 8)[:, :8], o.decrypt(xo, 8)[:, :8], atol=1e-9)


def test_rotate_hoisted_bit_exact(edl):
    """Hoisted rotations (one modulus raise, several Galois elements) == the oracle's
    rotate_hoisted on every residue; rotation 0 is a copy."""
    from oracle import galois
    g, o = _pair(edl, logn=10, bits=[60, 40, 40, 40, 40, 60], seed=1)
    rs = [1, -2, 5, 0]
    g.galois_keygen(7, [r for r in rs if r])
    gk = {galois.galois_element(r, o.n): galois.galois_keygen(o, 7, galois.galois_element(r, o.n)) for r in rs if r}
    lvl = 3
    X = ock.CtArray(_rand_ct(o, 3, lvl, 81), lvl, 2.0 ** 40, o.key_id)
    got = g.rotate_hoisted(_to_gpu(g, X.data, lvl, X.scale, o.key_id), rs)
    want = galois.rotate_hoisted(o, X, [r for r in rs if r], gk)
    for y, w in zip(got[:3], want):
        assert y.level == w.level and np.array_equal(y.numpy(g.n), w.data)
    assert np.array_equal(got[3].numpy(g.n), X.data)


def test_pt_mac_multi_bit_exact(c1pair):
    """edl_ct_pt_mac_multi == the oracle's sum over t of plaintext products (every limb
    path: q0 with 128-bit sums, the 40-bit limbs with FP64-pipe products), incl. all-(q-1)."""
    from oracle import galois
    g, o = c1pair
    lvl, T, F, n = 4, 3, 2, 2
    rots = _rand_ct(o, T * n, lvl, 91)
    rots[0] = np.stack([np.stack([np.full(o.n, o.q[i] - 1, dtype=np.uint64) for i in range(lvl + 1)])] * 2)
    pts = random_residues((F, T, lvl + 1, o.n), o.q[: lvl + 1] * (F * T), seed=92)
    pts[0, 0] = np.stack([np.full(o.n, o.q[i] - 1, dtype=np.uint64) for i in range(lvl + 1)])
    rg = _to_gpu(g, rots, lvl, 2.0 ** 40, o.key_id)
    ptg = g.torch.from_numpy(pts.view(np.int64).reshape(-1).copy()).cuda()
    got = g.pt_mac_multi(rg, T, ptg, F, lvl, 2.0 ** 20)
    assert got.count == n * F and got.scale == 2.0 ** 60
    R = rots.reshape(T, n, 2, lvl + 1, o.n)
    for c in range(n):
        for f in range(F):
            acc = None
            for t in range(T):
                y = galois.mul_plain(o, ock.CtArray(R[t, c:c + 1], lvl, 2.0 ** 40, o.key_id), pts[f, t][None], 2.0 ** 20)
                acc = y if acc is None else o.add(acc, y)
            assert np.array_equal(got.numpy(g.n)[c * F + f], acc.data[0])


def test_mul_relin_mixed_levels(c0pair):
    g, o = c0pair
    A = ock.CtArray(_rand_ct(o, 2, 2, 41), 2, 2.0 ** 40, o.key_id)
    B = ock.CtArray(_rand_ct(o, 2, 1, 42), 1, 2.0 ** 40, o.key_id)
    got = g.mul_relin(_to_gpu(g, A.data, 2, A.scale, o.key_id), _to_gpu(g, B.data, 1, B.scale, o.key_id))
    assert got.level == 1
    assert np.array_equal(got.numpy(g.n), o.mul_relin(A, B).data)


# ---------------------------------------------------------------- layers
def test_layers_small_bit_exact(c1pair):
    """CC (8x8 image, 2 filters) -> sigma_a -> dense 8->3 on ciphertexts encrypted by both sides."""
    g, o = c1pair
    rng = np.random.default_rng(0)
    B = 8192
    imgs = rng.integers(0, 256, (B, 8, 8)) / 255.0
    K, kb = rng.normal(0, 0.1, (2, 4, 4)), rng.normal(0, 0.1, 2)
    W, b = rng.normal(0, 0.1, (3, 8)), rng.normal(0, 0.1, 3)
    polys = np.stack([o.encode(v) for v in imgs.reshape(B, 64).T])
    xo = o.encrypt_poly(polys, 2, 0, o.p.scale)
    xg = g.encrypt_poly(polys, scale=o.p.scale, enc_seed=2)
    cc_o = olay.cross_correlate(o, xo, 8, 8, K, 4, kb)
    cc_g = g.cross_correlate(xg, 8, 8, K, 4, kb)
    assert cc_g.scale == cc_o.scale and np.array_equal(cc_g.numpy(g.n), cc_o.data)
    act_o = olay.poly_activation(o, cc_o, onet.SIGMA_A)
    act_g = g.poly_activation(cc_g, onet.SIGMA_A)
    assert act_g.level == act_o.level and act_g.scale == act_o.scale
    assert np.array_equal(act_g.numpy(g.n), act_o.data)
    out_o = olay.dense(o, act_o, W, b)
    out_g = g.dense(act_g, W, b)
    assert np.array_equal(out_g.numpy(g.n), out_o.data)
    want = onet.sigma_a(onet.cc_float64(imgs, K, kb)) @ W.T + b
    assert np.max(np.abs(g.decrypt(out_g, B).T - want)) < 1e-3


def test_mac_layers_extreme_residues(c1pair):
    """CC and dense MACs on ciphertexts whose residues are all q_i - 1 (the largest operands
    of every arithmetic path: FP64-pipe products and sums on the 40-bit limbs, 128-bit sums
    on q0), GPU == oracle on every residue."""
    g, o = c1pair
    lvl = o.L
    data = np.zeros((64, 2, lvl + 1, o.n), dtype=np.uint64)
    for i in range(lvl + 1):
        data[:, :, i, :] = np.uint64(o.q[i] - 1)
    xo = ock.CtArray(data, lvl, 2.0 ** 40, o.key_id)
    xg = _to_gpu(g, data, lvl, 2.0 ** 40, o.key_id)
    rng = np.random.default_rng(21)
    K, kb = rng.normal(0, 0.5, (3, 4, 4)), rng.normal(0, 0.1, 3)
    cc_o = olay.cross_correlate(o, xo, 8, 8, K, 4, kb)
    cc_g = g.cross_correlate(xg, 8, 8, K, 4, kb)
    assert np.array_equal(cc_g.numpy(g.n), cc_o.data)
    W, b = rng.normal(0, 0.5, (5, cc_o.count)), rng.normal(0, 0.1, 5)
    assert np.array_equal(g.dense(cc_g, W, b).numpy(g.n), olay.dense(o, cc_o, W, b).data)
    # key switch (+ fused rescale epilogues) on the same extreme operands
    A = ock.CtArray(data[:2, :, :lvl].copy(), lvl - 1, 2.0 ** 40, o.key_id)
    Ag = _to_gpu(g, A.data, lvl - 1, 2.0 ** 40, o.key_id)
    m_o = o.mul_relin(A, A)
    m_g = g.mul_relin(Ag, Ag)
    assert np.array_equal(m_g.numpy(g.n), m_o.data)
    assert np.array_equal(g.rescale(m_g).numpy(g.n), o.rescale(m_o).data)


@pytest.mark.parametrize("H,F,kh,stride,ksd", [(10, 11, 4, 2, 0.3), (12, 3, 4, 4, 3.0), (9, 4, 3, 3, 0.3)])
def test_cc_geometries(c1pair, H, F, kh, stride, ksd):
    """Cross-correlation beyond C1's geometry, GPU == oracle on every residue: more filters
    than one launch chunk (11 = 8 + 3), overlapping windows (stride 2 < 4), a 3x3 kernel
    (k_cc_mac2 path; 4x4 kernels take k_cc_mac4), and weights ~N(0, 3) (integer encodings
    past 2^40: large 128-bit sums on q0)."""
    g, o = c1pair
    lvl = o.L
    rng = np.random.default_rng(100 + H)
    data = _rand_ct(o, H * H, lvl, 101 + H)
    xo = ock.CtArray(data, lvl, 2.0 ** 40, o.key_id)
    xg = _to_gpu(g, data, lvl, 2.0 ** 40, o.key_id)
    K, kb = rng.normal(0, ksd, (F, kh, kh)), rng.normal(0, 0.1, F)
    cc_o = olay.cross_correlate(o, xo, H, H, K, stride, kb)
    cc_g = g.cross_correlate(xg, H, H, K, stride, kb)
    assert cc_g.count == cc_o.count and np.array_equal(cc_g.numpy(g.n), cc_o.data)


def test_dense_ragged_and_deferred(c1pair):
    """Dense with K > 256 (accumulator folding), O > 16 (several output chunks), and the
    C4 deferred-rescale + uint64 combine + mod_reduce path (O15)."""
    g, o = c1pair
    lvl, K, O = 2, 300, 19
    X = ock.CtArray(_rand_ct(o, K, lvl, 51), lvl, 2.0 ** 40, o.key_id)
    W = np.random.default_rng(1).normal(0, 0.1, (O, K))
    xg = _to_gpu(g, X.data, lvl, X.scale, o.key_id)
    assert np.array_equal(g.dense(xg, W, None).numpy(g.n), olay.dense(o, X, W, None).data)
    full = olay.dense_partial(o, X, W)
    parts = []
    for r in range(3):
        sl = list(range(r * K // 3, (r + 1) * K // 3))
        parts.append(g.dense(_to_gpu(g, X.data[sl], lvl, X.scale, o.key_id), W[:, sl], None, defer_rescale=True))
    acc = parts[0]
    acc.tensor = parts[0].tensor + parts[1].tensor + parts[2].tensor      # int64 add == uint64 wrap
    g.mod_reduce(acc)
    assert np.array_equal(acc.numpy(g.n), full.data)
    b = np.arange(O) * 0.01
    assert np.array_equal(g.dense_finish(acc, b).numpy(g.n), olay.dense_finish(o, full, b).data)


def test_c0_end_to_end(c0pair):
    from paper_2110_13638_b200.networks import C0Net
    g, o = c0pair
    inp = c0_inputs()
    polys = np.stack([o.encode(v) for v in inp.X.T])
    xo = o.encrypt_poly(polys, 2, 0, o.p.scale)
    xg = g.encrypt_poly(polys, scale=o.p.scale, enc_seed=2)
    ro = onet.c0_forward(o, xo, inp.W, inp.b)
    rg = C0Net(g, inp.W, inp.b).forward(xg, keep=True)
    assert np.array_equal(rg["dense"].numpy(g.n), ro["dense"].data)
    assert np.array_equal(rg["out"].numpy(g.n), ro["out"].data)
    got = g.decrypt(rg["out"], 64).T
    assert np.max(np.abs(got - onet.c0_float64(inp.X, inp.W, inp.b))) < 1e-3


# ---------------------------------------------------------------- errors / edge cases
def test_errors_and_empty(edl, c0pair):
    g, o = c0pair
    A = _to_gpu(g, _rand_ct(o, 2, 0, 61), 0, 2.0 ** 40, o.key_id)
    with pytest.raises(edl.LevelError):
        g.rescale(A)
    B = _to_gpu(g, _rand_ct(o, 2, 0, 62), 0, 2.0 ** 41, o.key_id)
    with pytest.raises(edl.ScaleError):
        g.add(A, B)
    C = _to_gpu(g, _rand_ct(o, 2, 0, 63), 0, 2.0 ** 40, o.key_id + 99)
    with pytest.raises(edl.KeyMismatch):
        g.add(A, C)
    D = _to_gpu(g, _rand_ct(o, 3, 0, 64), 0, 2.0 ** 40, o.key_id)
    with pytest.raises(edl.ShapeMismatch):
        g.add(A, D)
    with pytest.raises(edl.CapacityError):
        g.encode(np.zeros((1, 4097)))
    with pytest.raises(edl.ArgError):
        g.poly_activation(_to_gpu(g, _rand_ct(o, 1, 2, 65), 2, 2.0 ** 40, o.key_id), (1, 2, 3, 4, 5))
    E = g.empty(0, 2)
    E.key_id, E.scale = o.key_id, 2.0 ** 40
    assert g.add(E, E).count == 0
    assert g.rescale(E).count == 0
    # empty batches through every batched entry point of the hot path and the wire formats
    assert g.mul_relin(E, E).count == 0
    assert g.poly_activation(E, (0.5, 0.197, 0.0, -0.004)).count == 0
    assert g.pt_mul(E, np.zeros(0), 2.0 ** 20).count == 0
    assert g.packed_bytes(0, 2) == 0 and g.seeded_bytes(0, 2) == 0
    assert g.encrypt_poly_sk(np.zeros((0, g.n), dtype=np.int64), scale=2.0 ** 40, enc_seed=1).count == 0
    wire = g.torch.empty(0, dtype=g.torch.int64, device="cuda")
    assert g.unpack_seeded(wire, 0, 2, 2.0 ** 40, o.key_id, enc_seed=1).count == 0


@pytest.mark.parametrize("which", ["linear", "relu_a"])
def test_linear_and_relu_activations_bit_exact(c1pair, which):
    """NEXT f2: the paper's linear sigmoid and ReLU_a schedules, GPU residues == oracle,
    decrypted values == float64 polynomial within 1e-3."""
    from oracle import networks as onet
    g, o = c1pair
    z = random_slots(3, 8192, seed=11, lo=-1, hi=1)
    polys = np.stack([o.encode(v) for v in z])
    xo = o.encrypt_poly(polys, enc_seed=2, obj0=0, scale=o.p.scale)
    xg = g.encrypt_poly(polys, scale=o.p.scale, enc_seed=2)
    cf = onet.SIGMA_LINEAR if which == "linear" else onet.relu_a_coeffs(1.0)
    got, want = g.poly_activation(xg, cf), olay.poly_activation(o, xo, cf)
    assert got.level == want.level and got.scale == want.scale
    assert np.array_equal(got.numpy(g.n), want.data)
    ref = 0.5 + 0.197 * z if which == "linear" else onet.relu_a(z, 1.0)
    assert np.max(np.abs(g.decrypt(got, 8192) - ref)) < 1e-3


@pytest.mark.parametrize("coeffs", ["relu_a", "sigma_a"])
def test_activations_two_stream_batches(c0pair, coeffs):
    """Batches large enough for the two-stream schedules (key switches split in halves,
    sigma's scalar rescales on the side stream, fused output assembly): 34 ciphertexts,
    GPU == oracle on every residue (N=2^13, level 2)."""
    from oracle import networks as onet
    g, o = c0pair
    lvl, cnt = 2, 34
    A = ock.CtArray(_rand_ct(o, cnt, lvl, 71), lvl, 2.0 ** 40, o.key_id)
    cf = onet.relu_a_coeffs(1.0) if coeffs == "relu_a" else onet.SIGMA_A
    got = g.poly_activation(_to_gpu(g, A.data, lvl, A.scale, o.key_id), cf)
    want = olay.poly_activation(o, A, cf)
    assert got.level == want.level and got.scale == want.scale
    assert np.array_equal(got.numpy(g.n), want.data)


def _host_pack(data, qs, n):
    """Independent numpy packer of the wire format (edl.h): limb i's residues in bits(q_i)
    bits, little-endian, coefficient k at bit k*bits."""
    out = []
    cnt, two, nl, _ = data.shape
    for c in range(cnt):
        for p in range(two):
            for i in range(nl):
                b = int(qs[i]).bit_length()
                acc = 0
                for k, v in enumerate(data[c, p, i].tolist()):
                    acc |= int(v) << (k * b)
                words = n * b // 64
                out.extend((acc >> (64 * w)) & ((1 << 64) - 1) for w in range(words))
    return np.array(out, dtype=np.uint64)


@pytest.mark.parametrize("level", [0, 2, 4])
def test_wire_format_pack_unpack(c1pair, level):
    """Packed transfer format: device pack == independent host packing of the same
    residues, unpack(pack(x)) == x, and the size is 27.5/40 of the 64-bit layout at L=4."""
    g, o = c1pair
    A = _rand_ct(o, 3, level, 70 + level)
    x = _to_gpu(g, A, level, 2.0 ** 40, o.key_id)
    nbytes = g.packed_bytes(3, level)
    assert nbytes == 3 * 2 * sum(g.n * int(q).bit_length() // 8 for q in o.q[: level + 1])
    packed = g.pack(x)
    assert packed.numel() * 8 == nbytes
    host = packed.cpu().numpy().view(np.uint64)
    if level == 0:   # the pure-Python packer is slow; pin the bit layout on the smallest case
        assert np.array_equal(host, _host_pack(A, o.q, g.n))
    y = g.unpack(packed, 3, level, 2.0 ** 40, o.key_id)
    assert y.level == level and y.count == 3 and y.scale == 2.0 ** 40
    assert np.array_equal(y.numpy(g.n), A)


def test_host_wire_path(c1pair):
    """C-ABI host-buffer path (edl_wire_upload / edl_cts_unpack_host / edl_cts_unpack_seeded_host /
    edl_cts_download / edl_ctx_sync): wire bytes in pinned HOST memory -> device array ==
    the oracle's residues, for both slots, slot reuse without synchronisation in between,
    public-key and seeded secret-key formats; downloaded bytes == the device array; errors."""
    import torch
    g, o = c1pair
    lvl = 3
    A = [_rand_ct(o, 3, lvl, 170 + k) for k in range(3)]
    hosts = []
    for a_ in A:
        dev = g.pack(_to_gpu(g, a_, lvl, 2.0 ** 40, o.key_id))
        h = torch.empty(dev.numel(), dtype=torch.int64, pin_memory=True)
        h.copy_(dev.cpu())
        hosts.append(h)
    outs = []
    for k, h in enumerate(hosts):               # slots 0, 1, 0: the third upload reuses slot 0
        g.wire_upload(k % 2, h)
        outs.append(g.unpack_host(k % 2, 3, lvl, 2.0 ** 40, o.key_id))
    back = torch.empty(outs[2].tensor.numel(), dtype=torch.int64, pin_memory=True)
    g.download(outs[2], back)
    g.sync()
    for a_, y in zip(A, outs):
        assert y.count == 3 and y.level == lvl and np.array_equal(y.numpy(g.n), a_)
    assert np.array_equal(back.numpy().view(np.uint64).reshape(A[2].shape), A[2])
    # seeded secret-key wire: c0 from the host, c1 regenerated on the device
    polys = np.random.default_rng(23).integers(-2 ** 40, 2 ** 40, (2, o.n))
    xs = g.encrypt_poly_sk(polys, scale=2.0 ** 40, enc_seed=9, obj0=4)
    c0 = g.pack_c0(xs)
    hc = torch.empty(c0.numel(), dtype=torch.int64, pin_memory=True)
    hc.copy_(c0.cpu())
    g.wire_upload(1, hc)
    ys = g.unpack_seeded_host(1, 2, xs.level, xs.scale, xs.key_id, enc_seed=9, obj0=4)
    g.sync()
    assert np.array_equal(ys.numpy(g.n), o.encrypt_poly_sk(polys, enc_seed=9, obj0=4, scale=2.0 ** 40).data)
    # a slot holding fewer bytes than the array needs, and a bad slot
    g.wire_upload(0, hc)
    with pytest.raises(Exception):
        g.unpack_host(0, 3, lvl, 2.0 ** 40, o.key_id)
    with pytest.raises(Exception):
        g.wire_upload(2, hc)


# ---------------------------------------------------------------- NEXT f1: rotations, plaintext vectors
@pytest.fixture(scope="module")
def f1pair(c1pair):
    from oracle import galois as og
    g, o = c1pair
    steps = [1, 2, 8, 16, -2, 28]
    g.galois_keygen(7, steps)
    gk = {og.galois_element(r, o.n): og.galois_keygen(o, 7, og.galois_element(r, o.n)) for r in steps}
    return g, o, gk


def test_galois_key_bit_exact(f1pair):
    from oracle import galois as og
    g, o, gk = f1pair
    assert np.array_equal(g.export_galois_key(1), gk[og.galois_element(1, o.n)])


@pytest.mark.parametrize("r", [1, -2, 28])
def test_rotate_bit_exact(f1pair, r):
    from oracle import galois as og
    g, o, gk = f1pair
    lvl = 3
    A = ock.CtArray(_rand_ct(o, 2, lvl, 90 + r), lvl, 2.0 ** 40, o.key_id)
    got = g.rotate(_to_gpu(g, A.data, lvl, A.scale, o.key_id), r)
    want = og.rotate(o, A, r, gk)
    assert got.level == lvl and got.scale == A.scale
    assert np.array_equal(got.numpy(g.n), want.data)


def test_plain_vector_product_bit_exact(f1pair):
    from oracle import galois as og
    g, o, _ = f1pair
    w = np.random.default_rng(5).uniform(-1, 1, 784)
    lvl = 4
    pt_o = og.encode_plain(o, w, float(o.q[lvl]), lvl)
    pt_g = g.encode_pt_poly(o.encode(w, float(o.q[lvl]))[None, :], lvl)   # same integer poly (Z1)
    pt_h = g.encode_pt(w, float(o.q[lvl]), lvl)                           # library host encoder
    assert pt_h.numel() == pt_g.numel()
    assert np.array_equal(pt_g.cpu().numpy().view(np.uint64).reshape(pt_o.shape), pt_o)
    A = ock.CtArray(_rand_ct(o, 3, lvl, 95), lvl, 2.0 ** 40, o.key_id)
    got = g.pt_vec_mul(_to_gpu(g, A.data, lvl, A.scale, o.key_id), pt_g, 1, lvl, float(o.q[lvl]))
    want = og.mul_plain(o, A, np.broadcast_to(pt_o, (3,) + pt_o.shape), float(o.q[lvl]))
    assert got.scale == want.scale
    assert np.array_equal(got.numpy(g.n), want.data)


def test_masked_cc_bit_exact_and_float64(f1pair):
    """The paper's one-image-per-ciphertext CC (kernel masquerading + rotation window sums)
    on 8x8 images, 2 filters 4x4 stride 4: GPU residues == oracle, anchors == float64."""
    from oracle import galois as og, networks as onet
    from paper_2110_13638_b200 import masquerade
    g, o, gk = f1pair
    rng = np.random.default_rng(6)
    imgs = rng.integers(0, 256, (2, 8, 8)) / 255.0
    K, kb = rng.normal(0, 0.1, (2, 4, 4)), rng.normal(0, 0.1, 2)
    assert np.array_equal(masquerade.masquerade_masks(K, 8, 8, 4), og.masquerade_masks(K, 8, 8, 4))
    polys = np.stack([o.encode(v) for v in imgs.reshape(2, 64)])
    xo = o.encrypt_poly(polys, enc_seed=2, obj0=0, scale=o.p.scale)
    xg = g.encrypt_poly(polys, scale=o.p.scale, enc_seed=2)
    yg = masquerade.masked_cc(g, xg, K, 8, 8, 4, kb, encode=lambda z, sc: o.encode(z, sc))
    yo = og.masked_cc(o, xo, K, 8, 8, 4, kb, gk)
    assert yg.count == 4 and yg.level == yo.level
    assert np.array_equal(yg.numpy(g.n), yo.data)
    dec = g.decrypt(yg, 64).reshape(2, 2, 64)
    want = onet.cc_float64(imgs, K, kb)
    anchors = masquerade.anchor_slots(8, 8, 4, 4, 4)
    for b in range(2):
        for f in range(2):
            assert np.max(np.abs(dec[b, f, anchors] - want[b, f * 4:(f + 1) * 4])) < 1e-4



# ---------------------------------------------------------------- NEXT f3: device encode / decode
@pytest.mark.parametrize("logn", [10, 11, 13, 14, 15, 16])
def test_device_encode_contract(edl, logn):
    """Device canonical embedding vs the oracle encoder: the +-1 contract (reading Z1), at
    every row length of the four-step FFT (N/128 = 8 .. 512)."""
    from oracle import encoding
    if logn in (13, 14):
        g = edl.Context(edl.params_from_depth(2 if logn == 13 else 4))
    else:
        g = edl.Context(edl.params_from_bits(logn, [60, 40, 60]))
    z = random_slots(3, 1 << (logn - 1), seed=logn, lo=-1, hi=1)
    got = g.encode_device(z, 2.0 ** 40).cpu().numpy()
    want = np.stack([encoding.encode(v, 1 << logn, 2.0 ** 40) for v in z])
    d = np.abs(got - want)
    assert d.max() <= 1 and (d > 0).mean() <= 0.01


def test_device_round_trip_and_decrypt(c1pair):
    """encode_device -> encrypt_poly -> (ops) -> decrypt_device matches the host decrypt
    and the slots."""
    g, o = c1pair
    z = random_slots(4, 8192, seed=8, lo=-1, hi=1)
    polys = g.encode_device(z, o.p.scale)
    x = g.encrypt_poly(polys, scale=o.p.scale, enc_seed=2)
    dev = g.decrypt_device(x, 8192).cpu().numpy()
    assert np.max(np.abs(dev - z)) < 1e-6
    assert np.max(np.abs(dev - g.decrypt(x, 8192))) < 1e-9
    y = g.rescale(g.mul_relin(x, x))                              # multi-limb CRT lift, level 3
    assert np.max(np.abs(g.decrypt_device(y, 8192).cpu().numpy() - z * z)) < 1e-5
    r = g.rescale(g.rescale(g.rescale(y)))                        # level 0: single-limb lift
    hd, dd = g.decrypt(r, 100), g.decrypt_device(r, 100).cpu().numpy()   # (scale ~1e-24: large values)
    assert np.max(np.abs(dd - hd) / np.maximum(1.0, np.abs(hd))) < 1e-9


def test_keygen_drops_galois_keys(edl):
    """a second keygen must not leave Galois keys of the old secret in place."""
    g, o = _pair(edl, depth=2)
    g.galois_keygen(5, [1])
    g.keygen(3)
    X = _rand_ct(o, 1, 2, 91)
    with pytest.raises(edl.EdlError):
        g.rotate(_to_gpu(g, X, 2, 2.0 ** 40, g.key_id), 1)


def test_chunked_keyswitch_bit_exact(edl, monkeypatch):
    """Key switches in L2-sized chunks over the two streams (EDL_KS_CHUNK): 37 ciphertexts
    (ragged last chunk) at every level of the C0 chain, and the sigma_a-shaped x^2 layer,
    against the oracle."""
    monkeypatch.setenv("EDL_KS_CHUNK", "8")
    g, o = _pair(edl, depth=2)
    for lvl in (1, 2):
        A = ock.CtArray(_rand_ct(o, 37, lvl, 151 + lvl), lvl, 2.0 ** 40, o.key_id)
        B = ock.CtArray(_rand_ct(o, 37, lvl, 161 + lvl), lvl, 2.0 ** 40, o.key_id)
        got = g.mul_relin(_to_gpu(g, A.data, lvl, A.scale, o.key_id), _to_gpu(g, B.data, lvl, B.scale, o.key_id))
        assert np.array_equal(got.numpy(g.n), o.mul_relin(A, B).data), lvl
    X = ock.CtArray(_rand_ct(o, 37, 2, 171), 2, 2.0 ** 40, o.key_id)
    got = g.poly_activation(_to_gpu(g, X.data, 2, X.scale, o.key_id), [0.0, 0.0, 1.0])
    assert np.array_equal(got.numpy(g.n), olay.poly_activation(o, X, [0.0, 0.0, 1.0]).data)


def test_fused_raise_bit_exact(edl, monkeypatch):
    """The fused d2 INTT + modulus raise (k_relin_raise, EDL_RAISE_FUSED=1) against the
    oracle: mul_relin at every level of the C1 chain (16 ciphertexts: both stream halves)
    and the sigma_a layer."""
    monkeypatch.setenv("EDL_RAISE_FUSED", "1")
    g, o = _pair(edl, depth=4)
    for lvl in (1, 2, 3, 4):
        A = ock.CtArray(_rand_ct(o, 16, lvl, 181 + lvl), lvl, 2.0 ** 40, o.key_id)
        B = ock.CtArray(_rand_ct(o, 16, lvl, 191 + lvl), lvl, 2.0 ** 40, o.key_id)
        got = g.mul_relin(_to_gpu(g, A.data, lvl, A.scale, o.key_id), _to_gpu(g, B.data, lvl, B.scale, o.key_id))
        assert np.array_equal(got.numpy(g.n), o.mul_relin(A, B).data), lvl
    X = ock.CtArray(_rand_ct(o, 3, 3, 199), 3, 2.0 ** 40, o.key_id)
    got = g.poly_activation(_to_gpu(g, X.data, 3, X.scale, o.key_id), [0.5, 0.197, 0.0, -0.004])
    assert np.array_equal(got.numpy(g.n), olay.poly_activation(o, X, [0.5, 0.197, 0.0, -0.004]).data)
