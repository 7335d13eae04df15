"""Oracle: the paper's layer nodes over ciphertext arrays (TEST INFRASTRUCTURE ONLY).

* cross_correlate  -- Eq. cnn, biased cross-correlation; in the
  batch-in-slots layout every kernel tap is a ct x scalar product (E3), the bias is
  added once after rescale (reading Z7).
* poly_activation  -- sigma_a(x) = 0.5 + 0.197x - 0.004x^3 (reading
  Z9) on the fixed 2-level schedule of O13, or x^2 (config C0).
* dense            -- PAPER.md:298-309 ("accept multiple cyphertexts ... summed across
  the first axis"): out_o = sum_i W[o,i] x_i + b_o.
* combine_partials -- O15: uint64 sum of per-rank partial dense accumulators then
  mod q (north_star's "NCCL uint64 sum ... followed by a per-limb mod-q reduction").
"""
from __future__ import annotations

from typing import List, Sequence

import numpy as np

from . import ring
from .ckks import CkksError, Context, CtArray, ShapeMismatch, const_int


def weighted_sum(ctx: Context, xs: CtArray, idx: Sequence[int], w: Sequence[float], pt_scale: float) -> np.ndarray:
    """sum_t xs[idx[t]] * (rint(w[t]*pt_scale) mod q_i), both polys, mod q_i, no rescale."""
    lvl = xs.level
    acc = np.zeros((2, lvl + 1, ctx.n), dtype=np.uint64)
    for t, k in enumerate(idx):
        kk = const_int(w[t], pt_scale)
        for c in range(2):
            for i in range(lvl + 1):
                q = ctx.q[i]
                acc[c, i] = ring.add(acc[c, i], ring.mul_scalar(xs.data[k, c, i].copy(), kk % q, q), q)
    return acc


def cross_correlate(ctx: Context, x: CtArray, H: int, W: int, K: np.ndarray, stride: int,
                    bias: np.ndarray) -> CtArray:
    """x: H*W ciphertexts, pixel-major (row r, col c at r*W+c).  K: [F][kh][kw].
    out[f,r,c] = Rescale(sum_{u,v} x[r*st+u, c*st+v] * const(K[f,u,v], q_l)) + const(b_f)."""
    F, kh, kw = K.shape
    if x.count != H * W:
        raise ShapeMismatch("x must hold H*W ciphertexts")
    Ho, Wo = (H - kh) // stride + 1, (W - kw) // stride + 1
    l = x.level
    if l < 1:
        raise CkksError("LevelExhausted")
    pt_scale = float(ctx.q[l])
    out = np.empty((F * Ho * Wo, 2, l + 1, ctx.n), dtype=np.uint64)
    for f in range(F):
        for r in range(Ho):
            for c in range(Wo):
                idx = [(r * stride + u) * W + (c * stride + v) for u in range(kh) for v in range(kw)]
                w = [K[f, u, v] for u in range(kh) for v in range(kw)]
                out[(f * Ho + r) * Wo + c] = weighted_sum(ctx, x, idx, w, pt_scale)
    acc = CtArray(out, l, x.scale * pt_scale, x.key_id)
    y = ctx.rescale(acc)
    return ctx.add_scalar(y, np.repeat(np.asarray(bias, dtype=np.float64), Ho * Wo))


def dense_partial(ctx: Context, x: CtArray, Wt: np.ndarray) -> CtArray:
    """Un-rescaled accumulators sum_i x_i * const(W[o,i], q_l) (scale x.scale*q_l)."""
    O, K = Wt.shape
    if x.count != K:
        raise ShapeMismatch("dense: K inputs required")
    l = x.level
    if l < 1:
        raise CkksError("LevelExhausted")
    pt_scale = float(ctx.q[l])
    out = np.empty((O, 2, l + 1, ctx.n), dtype=np.uint64)
    for o in range(O):
        out[o] = weighted_sum(ctx, x, range(K), Wt[o], pt_scale)
    return CtArray(out, l, x.scale * pt_scale, x.key_id)


def dense_finish(ctx: Context, acc: CtArray, bias) -> CtArray:
    y = ctx.rescale(acc)
    if bias is not None:
        y = ctx.add_scalar(y, np.asarray(bias, dtype=np.float64))
    return y


def dense(ctx: Context, x: CtArray, Wt: np.ndarray, bias) -> CtArray:
    return dense_finish(ctx, dense_partial(ctx, x, Wt), bias)


def combine_partials(ctx: Context, parts: List[CtArray]) -> CtArray:
    """O15: elementwise uint64 sum (wrapping) of partial accumulators, then mod q_i."""
    s = np.zeros_like(parts[0].data)
    for p in parts:
        s = s + p.data                      # numpy uint64 add wraps mod 2^64; here R*q < 2^63
    out = np.empty_like(s)
    for i in range(parts[0].level + 1):
        out[:, :, i] = ring.reduce(np.ascontiguousarray(s[:, :, i]), ctx.q[i])
    return CtArray(out, parts[0].level, parts[0].scale, parts[0].key_id)


def square(ctx: Context, y: CtArray) -> CtArray:
    """C0 activation x^2: Rescale(Relin(y (x) y))."""
    return ctx.rescale(ctx.mul_relin(y, y))


def sigmoid_approx(ctx: Context, y: CtArray, c0: float = 0.5, c1: float = 0.197, c3: float = -0.004) -> CtArray:
    """O13 schedule for c0 + c1 y + c3 y^3 on 2 levels (4 rescales, 2 relins per ct)."""
    l = y.level
    if l < 2:
        raise CkksError("LevelExhausted")
    ql = float(ctx.q[l])
    y2 = ctx.rescale(ctx.mul_relin(y, y))                                   # 1. scale S^2/q_l
    u = ctx.rescale(ctx.mul_scalar(y, [c3] * y.count, ql))                  # 2. scale (S*q_l)/q_l
    v = ctx.rescale(ctx.mul_relin(u, y2))                                   # 3. level l-2
    s3 = v.scale
    p1 = s3 * ql / y.scale                                                  # 4. chosen so S*p1/q_l ~ S3
    w = ctx.mod_drop(ctx.rescale(ctx.mul_scalar(y, [c1] * y.count, p1)), l - 2)
    out = ctx.add(v, w)                                                     # 5.
    return ctx.add_scalar(out, [c0] * y.count)


def linear_activation(ctx: Context, y: CtArray, c0: float, c1: float) -> CtArray:
    """c0 + c1 y on 1 level: Rescale(y x const(c1, q_l)) + c0 -- the paper's linear
    sigmoid 0.5 + 0.197x."""
    l = y.level
    if l < 1:
        raise CkksError("LevelExhausted")
    u = ctx.rescale(ctx.mul_scalar(y, [c1] * y.count, float(ctx.q[l])))
    return ctx.add_scalar(u, [c0] * y.count)


def quadratic_activation(ctx: Context, y: CtArray, c0: float, c1: float, c2: float) -> CtArray:
    """c0 + c1 y + c2 y^2 on 2 levels (the paper's ReLU approximation R_a):
      y2 = Rescale(Relin(y (x) y))                  level l-1, scale S2 = S^2/q_l
      a  = Rescale(y2 x const(c2, q_{l-1}))         level l-2, scale (S2 q_{l-1})/q_{l-1}
      b  = mod_drop(Rescale(y x const(c1, p1)))     level l-2, p1 = S2 q_l / S so S p1/q_l ~ S2
      out = a + b + c0"""
    l = y.level
    if l < 2:
        raise CkksError("LevelExhausted")
    ql, qlm1 = float(ctx.q[l]), float(ctx.q[l - 1])
    y2 = ctx.rescale(ctx.mul_relin(y, y))
    a = ctx.rescale(ctx.mul_scalar(y2, [c2] * y.count, qlm1))
    p1 = y2.scale * ql / y.scale
    b = ctx.mod_drop(ctx.rescale(ctx.mul_scalar(y, [c1] * y.count, p1)), l - 2)
    return ctx.add_scalar(ctx.add(a, b), [c0] * y.count)


def poly_activation(ctx: Context, y: CtArray, coeffs: Sequence[float]) -> CtArray:
    """Fixed schedules (SURVEY O13 + NEXT f2): x^2 (C0), degree 1 (linear sigmoid),
    degree 2 (ReLU_a), degree 3 with c2 = 0 (sigma_a)."""
    coeffs = list(coeffs)
    if len(coeffs) == 3 and coeffs[0] == 0.0 and coeffs[1] == 0.0 and coeffs[2] == 1.0:
        return square(ctx, y)
    if len(coeffs) == 2:
        return linear_activation(ctx, y, coeffs[0], coeffs[1])
    if len(coeffs) == 3:
        return quadratic_activation(ctx, y, coeffs[0], coeffs[1], coeffs[2])
    if len(coeffs) == 4 and coeffs[2] == 0.0:
        return sigmoid_approx(ctx, y, coeffs[0], coeffs[1], coeffs[3])
    raise CkksError("unsupported polynomial schedule")
