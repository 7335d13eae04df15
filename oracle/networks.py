"""Oracle: the hot-path networks C0/C1/C3 and their float64 references (O14; TEST INFRASTRUCTURE ONLY).

The paper fires its graph node by node (Alg. 1-5); on the chain graphs
of the configs that is exactly layer-after-layer evaluation in edge order, which is
what these functions do.  ``*_float64`` evaluate the SAME polynomial network (same
weights, sigma_a, no exact sigmoid) in plain numpy.
"""
from __future__ import annotations

from typing import Dict, Optional

import math

import numpy as np

from . import layers
from .ckks import Context, CtArray
from .params import params_from_depth

SIGMA_A = (0.5, 0.197, 0.0, -0.004)   # PAPER.md:407 (reading Z9)
SIGMA_LINEAR = (0.5, 0.197)           # PAPER.md:292 (linear part of sigma_a)


def relu_a_coeffs(q: float = 1.0):
    """R_a(x) = 4/(3 pi q) x^2 + x/2 + q/(3 pi) as (c0, c1, c2)."""
    return (q / (3.0 * math.pi), 0.5, 4.0 / (3.0 * math.pi * q))


def relu_a(x, q: float = 1.0):
    c0, c1, c2 = relu_a_coeffs(q)
    return c0 + c1 * x + c2 * x * x
SQUARE = (0.0, 0.0, 1.0)


def sigma_a(x):
    return 0.5 + 0.197 * x - 0.004 * x ** 3


# ---------------- C0: dense 16->4, x^2 ----------------
def c0_context(key_seed: int = 1) -> Context:
    return Context(params_from_depth(2)).keygen(key_seed)


def c0_forward(ctx: Context, x: CtArray, W, b) -> Dict[str, CtArray]:
    h = layers.dense(ctx, x, W, b)
    y = layers.poly_activation(ctx, h, SQUARE)
    return {"dense": h, "out": y}


def c0_float64(X, W, b):
    return (X @ W.T + b) ** 2


# ---------------- C1: CC 5x4x4/4 -> sigma_a -> dense 245->10 ----------------
def c1_context(key_seed: int = 1) -> Context:
    return Context(params_from_depth(4)).keygen(key_seed)


def c1_forward(ctx: Context, x: CtArray, K, kb, W, b) -> Dict[str, CtArray]:
    cc = layers.cross_correlate(ctx, x, 28, 28, K, 4, kb)
    act = layers.poly_activation(ctx, cc, SIGMA_A)
    out = layers.dense(ctx, act, W, b)
    return {"cc": cc, "act": act, "out": out}


def cc_float64(images, K, kb, stride=4):
    """images (B, H, W) -> (B, F*Ho*Wo), flattened f-major like the ciphertext order."""
    B, H, Wd = images.shape
    F, kh, kw = K.shape
    Ho, Wo = (H - kh) // stride + 1, (Wd - kw) // stride + 1
    out = np.zeros((B, F, Ho, Wo))
    for f in range(F):
        for r in range(Ho):
            for c in range(Wo):
                win = images[:, r * stride:r * stride + kh, c * stride:c * stride + kw]
                out[:, f, r, c] = np.einsum("buv,uv->b", win, K[f]) + kb[f]
    return out.reshape(B, -1)


def c1_float64(images, K, kb, W, b):
    h = sigma_a(cc_float64(images, K, kb))
    return h @ W.T + b


# ---------------- C3: dense 32->64 -> sigma_a -> dense 64->1 ----------------
def c3_context(key_seed: int = 1) -> Context:
    return Context(params_from_depth(4)).keygen(key_seed)


def c3_forward(ctx: Context, x: CtArray, W1, b1, W2, b2) -> Dict[str, CtArray]:
    h = layers.dense(ctx, x, W1, b1)
    a = layers.poly_activation(ctx, h, SIGMA_A)
    out = layers.dense(ctx, a, W2, b2)
    return {"dense1": h, "act": a, "out": out}


def c3_float64(X, W1, b1, W2, b2):
    return sigma_a(X @ W1.T + b1) @ W2.T + b2
