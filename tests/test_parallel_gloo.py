"""N>1 path on CPU: world_size-2 gloo run of the C4 sharding plan (paper_2110_13638_b200.
parallel) with the oracle doing each rank's arithmetic.  The uint64 all-reduce of the
rank partials followed by mod q must equal the unsharded dense accumulator bit-exactly
(O15), for a ring small enough to run in seconds."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2110_13638_b200.parallel import dense_columns, rank_windows, strip_pixels, WINDOWS


def test_rank_windows_cover_every_unit_once():
    for B in (1, 2, 3, 8):
        for R in (1, 2, 3, 4, 8):
            seen = np.zeros((B, WINDOWS), dtype=int)
            sizes = []
            for r in range(R):
                n = 0
                for b, (w0, w1) in enumerate(rank_windows(R, r, B)):
                    seen[b, w0:w1] += 1
                    n += w1 - w0
                sizes.append(n)
            assert (seen == 1).all()
            assert max(sizes) - min(sizes) <= 1


def test_strip_pixels_are_the_windows():
    px = strip_pixels(0, 49)
    assert sorted(px) == list(range(784))
    img = np.arange(784).reshape(28, 28)
    strip = np.array(px).reshape(4, 4 * 49)
    for k in range(49):
        r, c = divmod(k, 7)
        assert np.array_equal(strip[:, 4 * k:4 * k + 4], img[4 * r:4 * r + 4, 4 * c:4 * c + 4])
    assert dense_columns(3, 5) == [3, 4, 52, 53, 101, 102, 150, 151, 199, 200]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, batches, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import ckks, layers, networks
    from oracle.params import make_params
    ctx = ckks.Context(make_params(1024, [60, 40, 40, 40, 40, 60])).keygen(1)
    rng = np.random.default_rng(7)
    K, kb = rng.normal(0, 0.1, (5, 4, 4)), rng.normal(0, 0.1, 5)
    W = rng.normal(0, 0.1, (10, 245))
    parts = np.zeros((batches, 10, 2, 2, 1024), dtype=np.uint64)
    for b, (w0, w1) in enumerate(rank_windows(world, rank, batches)):
        if w1 == w0:
            continue
        imgs = np.random.default_rng(100 + b).integers(0, 256, (512, 784)) / 255.0
        px = strip_pixels(w0, w1)
        x = ctx.encrypt(imgs[:, px].T, enc_seed=2, obj0=0)
        cc = layers.cross_correlate(ctx, x, 4, 4 * (w1 - w0), K, 4, kb)
        act = layers.poly_activation(ctx, cc, networks.SIGMA_A)
        parts[b] = layers.dense_partial(ctx, act, W[:, dense_columns(w0, w1)]).data
    t = torch.from_numpy(parts.view(np.int64).copy())
    dist.all_reduce(t, op=dist.ReduceOp.SUM)                 # uint64 sum == int64 wrap-around sum
    summed = t.numpy().view(np.uint64).reshape(parts.shape)
    if rank == 0:
        red = np.empty_like(summed)
        for i in range(2):
            red[:, :, :, i] = summed[:, :, :, i] % np.uint64(ctx.q[i])
        q.put(red)
    dist.destroy_process_group()


@pytest.mark.timeout(600)
def test_gloo_world2_combine_matches_unsharded():
    from oracle import ckks, layers, networks
    from oracle.params import make_params
    batches, world = 2, 2
    mpctx = mp.get_context("spawn")
    q = mpctx.Queue()
    port = _free_port()
    procs = [mpctx.Process(target=_worker, args=(r, world, port, batches, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=500)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # unsharded reference: the full 28x28 CC per batch, same keys/weights/encryption rule
    ctx = ckks.Context(make_params(1024, [60, 40, 40, 40, 40, 60])).keygen(1)
    rng = np.random.default_rng(7)
    K, kb = rng.normal(0, 0.1, (5, 4, 4)), rng.normal(0, 0.1, 5)
    W = rng.normal(0, 0.1, (10, 245))
    for b in range(batches):
        imgs = np.random.default_rng(100 + b).integers(0, 256, (512, 784)) / 255.0
        # encrypt each pixel with the object id it gets on its rank (strip position),
        # so the two runs encrypt identical ciphertexts
        cts = np.zeros((784, 2, 5, 1024), dtype=np.uint64)
        for r in range(world):
            w0, w1 = rank_windows(world, r, batches)[b]
            if w1 == w0:
                continue
            px = strip_pixels(w0, w1)
            x = ctx.encrypt(imgs[:, px].T, enc_seed=2, obj0=0)
            cts[px] = x.data
        X = ckks.CtArray(cts, 4, ctx.p.scale, ctx.key_id)
        cc = layers.cross_correlate(ctx, X, 28, 28, K, 4, kb)
        act = layers.poly_activation(ctx, cc, networks.SIGMA_A)
        full = layers.dense_partial(ctx, act, W).data
        assert np.array_equal(got[b], full)
