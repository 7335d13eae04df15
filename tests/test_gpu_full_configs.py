"""Full-size parity at BASELINE.json's configs, in the launch configuration bench.py times.

C1 (784 pixel ciphertexts, 8192 images): every residue of every layer boundary equals
the oracle's (the oracle run takes about a minute on one core), decrypted logits lie
within 1e-3 of float64 plaintext inference, and argmax agrees on non-near-tie samples.
C3 (tabular, 2 slot-batches x 32 features): same checks, plus the MSE vs float64.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gpu():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2110_13638_b200 import edl
    return edl


@pytest.mark.timeout(900)
def test_c1_full_bit_exact(gpu):
    from oracle import layers, networks as onet
    from paper_2110_13638_b200.networks import C1Net
    from synth import c1_inputs, c1_slots

    inp = c1_inputs(8192)
    octx = onet.c1_context(1)
    ctx = gpu.Context(gpu.params_from_depth(4)).keygen(1)
    polys = np.stack([octx.encode(z) for z in c1_slots(inp.images)])
    xo = octx.encrypt_poly(polys, 2, 0, octx.p.scale)
    xg = ctx.encrypt_poly(polys, scale=octx.p.scale, enc_seed=2)
    assert np.array_equal(xg.numpy(ctx.n), xo.data)
    rg = C1Net(ctx, inp.K, inp.kb, inp.W, inp.b).forward(xg, keep=True)
    cc = layers.cross_correlate(octx, xo, 28, 28, inp.K, 4, inp.kb)
    assert np.array_equal(rg["cc"].numpy(ctx.n), cc.data)
    act = layers.poly_activation(octx, cc, onet.SIGMA_A)
    assert np.array_equal(rg["act"].numpy(ctx.n), act.data)
    out = layers.dense(octx, act, inp.W, inp.b)
    assert np.array_equal(rg["out"].numpy(ctx.n), out.data)
    assert rg["out"].scale == out.scale and rg["out"].level == out.level == 0
    got = ctx.decrypt(rg["out"], 8192).T                      # (8192, 10)
    ref = onet.c1_float64(inp.images, inp.K, inp.kb, inp.W, inp.b)
    assert np.max(np.abs(got - ref)) < 1e-3
    top2 = np.sort(ref, axis=1)[:, -2:]
    clear = (top2[:, 1] - top2[:, 0]) > 1e-3
    assert np.array_equal(got.argmax(1)[clear], ref.argmax(1)[clear])


@pytest.mark.timeout(900)
def test_c3_full_bit_exact(gpu):
    from oracle import networks as onet
    from paper_2110_13638_b200.networks import C3Net
    from synth import c3_inputs

    inp = c3_inputs()
    octx = onet.c3_context(1)
    ctx = gpu.Context(gpu.params_from_depth(4)).keygen(1)
    net = C3Net(ctx, inp.W1, inp.b1, inp.W2, inp.b2)
    preds, xgs, outs_o = [], [], []
    for bidx in range(2):                                    # reading Z12: 2 slot-batches
        Xb = inp.X[bidx * 8192:(bidx + 1) * 8192]
        polys = np.stack([octx.encode(z) for z in Xb.T])
        xo = octx.encrypt_poly(polys, 2, 32 * bidx, octx.p.scale)
        xg = ctx.encrypt_poly(polys, scale=octx.p.scale, enc_seed=2, obj0=32 * bidx)
        ro = onet.c3_forward(octx, xo, inp.W1, inp.b1, inp.W2, inp.b2)
        rg = net.forward(xg, keep=True)
        for k in ("dense1", "act", "out"):
            assert np.array_equal(rg[k].numpy(ctx.n), ro[k].data), k
        preds.append(ctx.decrypt(rg["out"], 8192)[0])
        xgs.append(xg)
        outs_o.append(ro["out"].data)
    # both slot-batches in one pass (sigma_a once over all hidden ciphertexts): same residues
    for og, oo in zip(net.forward_many(xgs), outs_o):
        assert np.array_equal(og.numpy(ctx.n), oo), "forward_many"
    pred = np.concatenate(preds)
    ref = onet.c3_float64(inp.X, inp.W1, inp.b1, inp.W2, inp.b2)[:, 0]
    assert np.max(np.abs(pred - ref)) < 1e-3
    assert float(np.mean((pred - ref) ** 2)) < 1e-8


@pytest.mark.timeout(900)
def test_c4_sharded_one_gpu_emulation(gpu):
    """C4 on one GPU: R = 2 ranks' partials computed one after the other through the
    per-rank driver (parallel.ShardedCNN), summed as uint64 (the NCCL all-reduce's
    arithmetic), then mod q + rescale + bias: every output residue equals the unsharded
    C1 network's, for B = 2 batches."""
    from paper_2110_13638_b200 import parallel
    from paper_2110_13638_b200.networks import C1Net
    from synth import c1_images, c1_slots, c1_weights

    ctx = gpu.Context(gpu.params_from_depth(4)).keygen(1)
    K, kb, W, b = c1_weights()
    B, R = 2, 2
    full = []
    for bi in range(B):
        polys = ctx.encode(c1_slots(c1_images(8192, 2110 + bi)))
        full.append(ctx.encrypt_poly(polys, scale=2.0 ** 40, enc_seed=2))
    want = [C1Net(ctx, K, kb, W, b).forward(full[bi])["out"].numpy(ctx.n) for bi in range(B)]
    total = None
    for r in range(R):
        sh = parallel.ShardedCNN(ctx, K, kb, W, b, R, r, B)
        assert sh.units in (49 * B // R, 49 * B // R + 1)
        x = parallel.rank_inputs(ctx, sh, full)
        part = torch.empty(sh.partials_words(), dtype=torch.int64, device="cuda")
        lvl, sc = sh.partials(x, part)
        total = part if total is None else total + part          # int64 wrap == uint64 sum
    sh0 = parallel.ShardedCNN(ctx, K, kb, W, b, R, 0, B)
    outs = sh0.finish(total, lvl, sc, batches=range(B))
    for bi in range(B):
        assert np.array_equal(outs[bi].numpy(ctx.n), want[bi]), bi


@pytest.mark.timeout(900)
def test_f1_masked_cnn_vs_float64(gpu):
    """NEXT f1: C1's CNN in the paper's own layout (one image per ciphertext, kernel
    masquerading, rotation sums) decrypts to the float64 logits within 1e-3."""
    from oracle import networks as onet
    from paper_2110_13638_b200 import masquerade
    from synth import c1_images, c1_weights

    ctx = gpu.Context(gpu.params_from_depth(4)).keygen(1)
    ctx.galois_keygen(7, masquerade.network_rotations(28, 28, 4, 4))
    K, kb, W, b = c1_weights()
    imgs = c1_images(3, 2110)
    x = ctx.encrypt(imgs.reshape(3, 784), enc_seed=2)
    out = masquerade.masked_cnn(ctx, x, K, kb, W, b)
    assert out.count == 30 and out.level == 0
    got = ctx.decrypt(out, 1)[:, 0].reshape(3, 10)
    ref = onet.c1_float64(imgs, K, kb, W, b)
    assert np.max(np.abs(got - ref)) < 1e-3
    # the class-packed dense (35 instead of 100 dense rotations per image), same logits
    ctx.galois_keygen(8, masquerade.packed_rotations(ctx.n // 2, 784))
    outp = masquerade.masked_cnn(ctx, x, K, kb, W, b, packed=True)
    assert outp.count == 6 and outp.level == 0
    gotp = masquerade.packed_logits(ctx, outp, 10, 784)
    assert np.max(np.abs(gotp - ref)) < 1e-3
    # CC from hoisted tap rotations (one modulus raise for the 15 rotations of an image)
    ctx.galois_keygen(9, [r for r in masquerade.tap_rotations(4, 4, 28) if r])
    outh = masquerade.masked_cnn(ctx, x, K, kb, W, b, packed=True, hoisted=True)
    assert np.max(np.abs(masquerade.packed_logits(ctx, outh, 10, 784) - ref)) < 1e-3


@pytest.mark.timeout(1200)
def test_c4_sharded_step_vs_oracle(gpu):
    """C4 through ShardedCNN.step for R = 2 ranks and B = 2 batches:
    each rank's step runs CC -> sigma_a -> dense partials on its own (window, batch) units,
    the all-reduce is an in-process uint64 sum of both ranks' partials (the NCCL SUM's
    arithmetic), and the batch each rank finishes equals the ORACLE's C1 output for that
    batch on every residue (not only the GPU's unsharded network)."""
    from oracle import networks as onet
    from paper_2110_13638_b200 import parallel
    from synth import c1_images, c1_slots, c1_weights

    octx = onet.c1_context(1)
    ctx = gpu.Context(gpu.params_from_depth(4)).keygen(1)
    K, kb, W, b = c1_weights()
    B, R = 2, 2
    full, want = [], []
    for bi in range(B):
        polys = np.stack([octx.encode(z) for z in c1_slots(c1_images(8192, 2110 + bi))])
        xo = octx.encrypt_poly(polys, 2, 784 * bi, octx.p.scale)          # distinct object ids per batch
        full.append(ctx.encrypt_poly(polys, scale=octx.p.scale, enc_seed=2, obj0=784 * bi))
        assert np.array_equal(full[bi].numpy(ctx.n), xo.data)
        want.append(onet.c1_forward(octx, xo, K, kb, W, b)["out"])
    shards = [parallel.ShardedCNN(ctx, K, kb, W, b, R, r, B) for r in range(R)]
    xs = [parallel.rank_inputs(ctx, sh, full) for sh in shards]
    # every rank's partials first (what the all-reduce would see), then each rank's step
    parts = []
    for sh, x in zip(shards, xs):
        t = torch.empty(sh.partials_words(), dtype=torch.int64, device="cuda")
        sh.partials(x, t)
        parts.append(t)
    got = {}
    for r, (sh, x) in enumerate(zip(shards, xs)):
        others = [parts[k] for k in range(R) if k != r]

        def all_reduce(t, others=others):
            for o in others:
                t.add_(o)                                                   # int64 wrap == uint64 sum

        pt = torch.empty(sh.partials_words(), dtype=torch.int64, device="cuda")
        got.update(sh.step(x, pt, all_reduce))
    assert sorted(got) == list(range(B))
    for bi in range(B):
        assert got[bi].level == want[bi].level == 0 and got[bi].scale == want[bi].scale
        assert np.array_equal(got[bi].numpy(ctx.n), want[bi].data), bi


@pytest.mark.timeout(900)
def test_f1_packed_hoisted_bit_exact_vs_oracle(gpu):
    """NEXT f1 in the paper's layout, bit-exact: the GPU's hoisted
    masked CC -> sigma_a -> class-packed dense (with the sigma(kb) compensation and the
    ct + plaintext-vector bias) equals the oracle twin (oracle/galois.py
    masked_cnn_packed) on every residue, 2 images at N = 2^10 (16 x 16 images, 2 filters,
    dense 32 -> 3), with the oracle's encoder feeding both sides' plaintexts (reading Z1)."""
    from oracle import ckks as ock, galois, networks as onet
    from oracle.params import make_params
    from paper_2110_13638_b200 import masquerade

    bits = [60, 40, 40, 40, 40, 60]
    octx = ock.Context(make_params(1024, bits)).keygen(1)
    ctx = gpu.Context(gpu.params_from_bits(10, bits)).keygen(1)
    H = Wd = 16
    rw = np.random.default_rng(41)
    K = rw.normal(0.0, 0.1, (2, 4, 4))
    kb = rw.normal(0.0, 0.1, 2)
    Wt = rw.normal(0.0, 0.1, (3, 32))
    b = rw.normal(0.0, 0.1, 3)
    imgs = np.random.default_rng(42).integers(0, 256, (2, H, Wd)) / 255.0
    rots = sorted(set([r for r in masquerade.tap_rotations(4, 4, Wd) if r] +
                      masquerade.packed_rotations(ctx.n // 2, H * Wd)))
    ctx.galois_keygen(7, rots)
    gk = {galois.galois_element(r, octx.n): galois.galois_keygen(octx, 7, galois.galois_element(r, octx.n))
          for r in rots}
    polys = np.stack([octx.encode(z) for z in imgs.reshape(2, -1)])
    xo = octx.encrypt_poly(polys, 2, 0, octx.p.scale)
    xg = ctx.encrypt_poly(polys, scale=octx.p.scale, enc_seed=2)
    want = galois.masked_cnn_packed(octx, xo, K, kb, Wt, b, H, Wd, 4, onet.SIGMA_A, gk, octx.encode)
    got = masquerade.masked_cnn(ctx, xg, K, kb, Wt, b, H=H, W=Wd, stride=4, encode=octx.encode, packed=True,
                                hoisted=True)
    assert got.count == want.count == 4 and got.level == want.level == 0
    assert np.array_equal(got.numpy(ctx.n), want.data)
    ref = onet.c1_float64(imgs, K, kb, Wt, b)
    assert np.max(np.abs(masquerade.packed_logits(ctx, got, 3, H * Wd) - ref)) < 1e-3


def test_two_contexts_in_flight_bit_exact(gpu):
    """bench.py's batches-in-flight pipeline: two contexts (same key seed, own stream pair and
    scratch) fed alternately without synchronisation give the residues of one context run
    alone (C3 net, 32 -> 64 -> 1, as the workload: every layer kind of the path but the CC)."""
    import torch
    from paper_2110_13638_b200.networks import C3Net
    from synth import c3_inputs

    inp = c3_inputs()
    pipe = []
    for i in range(2):
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            ctx = gpu.Context(gpu.params_from_depth(4), stream=st).keygen(1)
            x = ctx.encrypt(inp.X[i * 8192:(i + 1) * 8192].T, enc_seed=2, obj0=32 * i)
        st.synchronize()
        pipe.append((ctx, C3Net(ctx, inp.W1, inp.b1, inp.W2, inp.b2), x, st))
    alone = []
    for ctx, net, x, st in pipe:
        with torch.cuda.stream(st):
            alone.append(net.forward(x)["out"].numpy(ctx.n))
    outs = []
    for k in range(6):                       # 3 rounds, alternating, nothing waits in between
        ctx, net, x, st = pipe[k % 2]
        with torch.cuda.stream(st):
            outs.append(net.forward(x)["out"])
    torch.cuda.synchronize()
    for k, o in enumerate(outs):
        assert np.array_equal(o.numpy(pipe[k % 2][0].n), alone[k % 2]), k
    assert pipe[0][0].key_id == pipe[1][0].key_id
    for ctx, *_ in pipe:
        ctx.close()
