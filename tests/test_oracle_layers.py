"""Pins for oracle layers / networks (O13-O15): decrypted outputs vs float64 evaluation
of the same polynomial network, closed-form activation values, sharded combine."""
import json
import os

import numpy as np
import pytest

from oracle import ckks, layers, networks
from oracle.params import make_params
from synth import c0_inputs

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_activation_closed_forms():
    g = json.load(open(os.path.join(GOLD, "activations.json")))
    for x, y in g["sigma_a"]["values"]:
        assert abs(networks.sigma_a(x) - y) < 1e-12
    assert networks.SIGMA_A == (0.5, 0.197, 0.0, -0.004)
    for x, q, y in g["relu_a"]["values"]:
        assert abs(networks.relu_a(x, q) - y) < 5e-6          # golden value printed to 5 digits
    # R_a is a degree-2 polynomial with odd part x/2: R_a(x) - R_a(-x) = x for every q
    for q in (1.0, 5.0):
        for x in (0.3, 1.7, -2.2):
            assert abs(networks.relu_a(x, q) - networks.relu_a(-x, q) - x) < 1e-12
    # it meets max(0, x) within q/(3 pi) at x = +-q (R_a(+-q) = q (1/2 +- 1/2) + 5 q/(3 pi) - ... )
    assert abs(networks.relu_a(1.0, 1.0) - (4 / (3 * np.pi) + 0.5 + 1 / (3 * np.pi))) < 1e-12


def test_c0_network_vs_float64():
    inp = c0_inputs()
    ctx = networks.c0_context()
    x = ctx.encrypt(inp.X.T, enc_seed=2)               # 16 cts, 64 slots used
    res = networks.c0_forward(ctx, x, inp.W, inp.b)
    assert res["dense"].level == 1 and res["out"].level == 0
    got = ctx.decrypt(res["out"], 64).T                # (64, 4)
    want = networks.c0_float64(inp.X, inp.W, inp.b)
    assert np.max(np.abs(got - want)) < 1e-3


@pytest.fixture(scope="module")
def small_ctx():
    # depth-4 chain at a small ring degree: same schedule as C1, seconds on the CPU
    return ckks.Context(make_params(1024, [60, 40, 40, 40, 40, 60])).keygen(1)


def test_cc_sigma_dense_small_vs_float64(small_ctx):
    ctx = small_ctx
    rng = np.random.default_rng(0)
    B = 512
    imgs = rng.integers(0, 256, (B, 8, 8)) / 255.0
    K = rng.normal(0, 0.1, (2, 4, 4))
    kb = rng.normal(0, 0.1, 2)
    W = rng.normal(0, 0.1, (3, 8))
    b = rng.normal(0, 0.1, 3)
    x = ctx.encrypt(imgs.reshape(B, 64).T, enc_seed=2)
    cc = layers.cross_correlate(ctx, x, 8, 8, K, 4, kb)
    assert cc.count == 8 and cc.level == 3
    cc_f = networks.cc_float64(imgs, K, kb)
    assert np.max(np.abs(ctx.decrypt(cc, B).T - cc_f)) < 1e-4
    act = layers.poly_activation(ctx, cc, networks.SIGMA_A)
    assert act.level == 1
    assert np.max(np.abs(ctx.decrypt(act, B).T - networks.sigma_a(cc_f))) < 1e-4
    out = layers.dense(ctx, act, W, b)
    assert out.level == 0
    want = networks.sigma_a(cc_f) @ W.T + b
    assert np.max(np.abs(ctx.decrypt(out, B).T - want)) < 1e-3


def test_combine_partials_equals_unsharded(small_ctx):
    """O15: sum over rank partials (uint64, then mod q) == unsharded accumulator, bit-exact."""
    ctx = small_ctx
    rng = np.random.default_rng(1)
    x = ctx.encrypt(rng.uniform(0, 1, (8, 512)), enc_seed=2, level=1)
    W = rng.normal(0, 0.1, (3, 8))
    full = layers.dense_partial(ctx, x, W)
    for R in (1, 2, 4, 8):
        parts = []
        for r in range(R):
            sl = list(range(r * 8 // R, (r + 1) * 8 // R))
            parts.append(layers.dense_partial(ctx, x.select(sl), W[:, sl]))
        comb = layers.combine_partials(ctx, parts)
        assert np.array_equal(comb.data, full.data)


def test_square_activation(small_ctx):
    ctx = small_ctx
    z = np.random.default_rng(2).uniform(-1, 1, (2, 512))
    y = layers.poly_activation(ctx, ctx.encrypt(z, 2), networks.SQUARE)
    assert np.max(np.abs(ctx.decrypt(y, 512) - z ** 2)) < 1e-5


def test_unsupported_schedule(small_ctx):
    ctx = small_ctx
    y = ctx.encrypt(np.zeros((1, 4)), 2)
    with pytest.raises(ckks.CkksError):
        layers.poly_activation(ctx, y, (1.0, 2.0, 3.0, 4.0, 5.0))
    with pytest.raises(ckks.CkksError):
        layers.poly_activation(ctx, y, (1.0, 2.0, 3.0, 4.0))      # cubic with c2 != 0
    with pytest.raises(ckks.CkksError):                               # level exhausted
        layers.poly_activation(ctx, ctx.encrypt(np.zeros((1, 4)), 2, level=1), networks.relu_a_coeffs())


@pytest.mark.parametrize("which", ["linear", "relu_a"])
def test_linear_and_relu_activations_vs_float64(small_ctx, which):
    """NEXT f2: the paper's linear sigmoid and ReLU approximation
     schedules decrypt to the float64 polynomial within 1e-4."""
    ctx = small_ctx
    z = np.random.default_rng(3).uniform(-1, 1, (3, 512))
    y = ctx.encrypt(z, 2)
    if which == "linear":
        out = layers.poly_activation(ctx, y, networks.SIGMA_LINEAR)
        want = 0.5 + 0.197 * z
        assert out.level == y.level - 1
    else:
        out = layers.poly_activation(ctx, y, networks.relu_a_coeffs(1.0))
        want = networks.relu_a(z, 1.0)
        assert out.level == y.level - 2
    assert np.max(np.abs(ctx.decrypt(out, 512) - want)) < 1e-4