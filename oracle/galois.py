"""Oracle: Galois rotations and plaintext-vector products for the paper's own CNN layout
(kernel masquerading).  TEST INFRASTRUCTURE ONLY.

Background (not in the paper, which delegates to MS-SEAL): the automorphism
sigma_g : a(X) -> a(X^g) (g odd) maps a CKKS slot vector z to z rotated left by r when
g = 5^r mod 2N (slot j <-> zeta^{5^j}, O5).  A ciphertext (c0, c1) under s becomes
(sigma_g c0, sigma_g c1) under sigma_g s; switching sigma_g c1 back to s uses a Galois key
with the relinearisation key's digit structure (O11) and gadget term P sigma_g(s):
  gk_j[0][i] = -a_j s + e_j + delta_ij (P mod q_i) sigma_g(s),  gk_j[1][i] = a_j,
a_j ~ Philox uniform (tag 9, object 64 g + j, limb i), e_j ~ CBD (tag 10, object 64 g + j).
Every function follows the definition step by step (coefficient-domain automorphism,
then NTT); the GPU path permutes NTT-domain residues instead and shares nothing.
"""
from __future__ import annotations

from typing import Dict, Sequence

import numpy as np

from . import ring, sampling as smp
from .ckks import Context, CtArray, CkksError


def galois_element(r: int, n: int) -> int:
    """g = 5^r mod 2N: left rotation of the N/2 slots by r (negative r: right)."""
    return pow(5, r % (n // 2), 2 * n)


def automorphism_coeff(a: np.ndarray, g: int, q: int) -> np.ndarray:
    """Coefficient domain: X^j -> X^{j g mod 2N} with X^N = -1 (residues mod q)."""
    n = a.shape[-1]
    out = np.zeros(n, dtype=np.uint64)
    for j in range(n):
        e = (j * g) % (2 * n)
        v = int(a[j])
        if e >= n:
            e -= n
            v = (q - v) % q
        out[e] = v
    return out


def automorphism_ntt(ctx: Context, a_hat: np.ndarray, g: int, idx: Sequence[int]) -> np.ndarray:
    """sigma_g on NTT-domain rows [len(idx)][N] (modulus index idx[r] for row r)."""
    coeff = ctx.intt(a_hat.copy(), list(idx))
    rows = np.stack([automorphism_coeff(coeff[r], g, ctx.moduli[i]) for r, i in enumerate(idx)])
    return ctx.ntt(rows, list(idx))


def galois_keygen(ctx: Context, seed: int, g: int) -> np.ndarray:
    """Galois key for element g: [L+1 digits][2][L+2 limbs][N], NTT domain."""
    n, L = ctx.n, ctx.L
    all_idx = list(range(L + 2))
    s_g = automorphism_ntt(ctx, ctx.s_hat, g, all_idx)             # sigma_g(s), every limb incl. P
    gk = np.zeros((L + 1, 2, L + 2, n), dtype=np.uint64)
    for j in range(L + 1):
        obj = 64 * g + j
        ej_hat = ctx.signed_to_ntt(smp.cbd(n, seed, obj, smp.TAG_GK_E), all_idx)
        for i in all_idx:
            m = ctx.moduli[i]
            aj = smp.uniform(n, seed, obj, i, smp.TAG_GK_A, m)
            bj = ring.sub(ej_hat[i], ring.mul(aj, ctx.s_hat[i], m), m)
            if i == j:
                bj = ring.add(bj, ring.mul_scalar(s_g[i], ctx.P % m, m), m)
            gk[j, 0, i] = bj
            gk[j, 1, i] = aj
    return gk


def rotate(ctx: Context, ct: CtArray, r: int, gkeys: Dict[int, np.ndarray]) -> CtArray:
    """Slots rotated left by r: (sigma_g c0 + ks_0, ks_1), ks = keyswitch(sigma_g c1, gk_g)."""
    n = ctx.n
    g = galois_element(r, n)
    if g not in gkeys:
        raise CkksError(f"no Galois key for rotation {r}")
    lvl = ct.level
    idx = list(range(lvl + 1))
    out = np.empty_like(ct.data)
    for c in range(ct.count):
        c0 = automorphism_ntt(ctx, ct.data[c, 0], g, idx)
        c1 = automorphism_ntt(ctx, ct.data[c, 1], g, idx)
        ks = ctx.keyswitch(c1, lvl, gkeys[g])
        for i in idx:
            out[c, 0, i] = ring.add(c0[i], ks[0, i], ctx.q[i])
            out[c, 1, i] = ks[1, i]
    return CtArray(out, lvl, ct.scale, ct.key_id)


def rotate_hoisted(ctx: Context, ct: CtArray, rs: Sequence[int], gkeys: Dict[int, np.ndarray]):
    """Several rotations of the same ciphertexts sharing one modulus raise ("hoisting",
    background, not in the paper): the digits of c1 are raised once,
        a_j = INTT_{q_j}(c1_j),  x_{j,t} = NTT_t(a_j mod t)  for every target t (q_0..q_l, P),
    and rotation r (g = 5^r) applies sigma_g to the raised digits instead of to c1:
        acc_{c,t} = sum_j sigma_g(x_{j,t}) gk_j[c][t],  (ks_0, ks_1) = ModDown(acc),
        out = (sigma_g(c0) + ks_0, ks_1).
    sigma_g(x_{j,t}) is the raise of sigma_g(a_j) up to the lift of the negated
    coefficients, so the result differs from `rotate` in its noise only; it decrypts to
    the rotated slots.  Returns one CtArray per rotation."""
    n, lvl = ctx.n, ct.level
    idx = list(range(lvl + 1))
    targets = idx + [ctx.L + 1]
    outs = []
    raised = []
    for c in range(ct.count):
        a = ctx.intt(ct.data[c, 1].copy(), idx)
        raised.append(np.stack([np.stack([ctx.ntt(ring.reduce(a[j].copy(), ctx.moduli[t])[None, :], [t])[0]
                                          for t in targets]) for j in idx]))   # [j][t][N]
    for r in rs:
        g = galois_element(r, n)
        if g not in gkeys:
            raise CkksError(f"no Galois key for rotation {r}")
        key = gkeys[g]
        out = np.empty_like(ct.data)
        for c in range(ct.count):
            acc = np.zeros((2, len(targets), n), dtype=np.uint64)
            for ti, t in enumerate(targets):
                mt = ctx.moduli[t]
                for j in idx:
                    xg = automorphism_ntt(ctx, raised[c][j][ti][None, :], g, [t])[0]
                    for k in range(2):
                        acc[k, ti] = ring.add(acc[k, ti], ring.mul(xg, key[j, k, t], mt), mt)
            ks = ctx.mod_down(acc, lvl)
            c0 = automorphism_ntt(ctx, ct.data[c, 0], g, idx)
            for i in idx:
                out[c, 0, i] = ring.add(c0[i], ks[0, i], ctx.q[i])
                out[c, 1, i] = ks[1, i]
        outs.append(CtArray(out, lvl, ct.scale, ct.key_id))
    return outs


def encode_plain(ctx: Context, z: np.ndarray, scale: float, level: int) -> np.ndarray:
    """Plaintext vector z -> NTT-domain residues [level+1][N] (O5 encode, then NTT)."""
    m = ctx.encode(z, scale)
    return ctx.signed_to_ntt(m, list(range(level + 1)))


def mul_plain(ctx: Context, ct: CtArray, pt_hat: np.ndarray, pt_scale: float) -> CtArray:
    """ct_c <- ct_c (.) pt_c (NTT-domain pointwise, both polys); pt_hat [count][L'+1][N]
    with L' >= ct.level; no rescale (O10 with a vector plaintext)."""
    out = np.empty_like(ct.data)
    for c in range(ct.count):
        for k in range(2):
            for i in range(ct.level + 1):
                out[c, k, i] = ring.mul(ct.data[c, k, i], pt_hat[c, i], ctx.q[i])
    return CtArray(out, ct.level, ct.scale * pt_scale, ct.key_id)


def masquerade_masks(K: np.ndarray, H: int, W: int, stride: int) -> np.ndarray:
    """Kernel masquerading (SPEC masquerade_kernel) for non-overlapping
    windows: one H*W mask per filter holding K[f] at every window position."""
    F, kh, kw = K.shape
    Ho, Wo = (H - kh) // stride + 1, (W - kw) // stride + 1
    masks = np.zeros((F, H * W))
    for f in range(F):
        for r in range(Ho):
            for c in range(Wo):
                for u in range(kh):
                    for v in range(kw):
                        masks[f, (r * stride + u) * W + c * stride + v] += K[f, u, v]
    return masks


def window_rotations(kh: int, kw: int, W: int):
    """Rotations that sum a kh x kw window into its top-left slot (power-of-two sizes)."""
    out = []
    s = 1
    while s < kw:
        out.append(s)
        s *= 2
    s = 1
    while s < kh:
        out.append(s * W)
        s *= 2
    return out


def masked_cc(ctx: Context, x: CtArray, K: np.ndarray, H: int, W: int, stride: int, bias, gkeys) -> CtArray:
    """The paper's CC on one-image-per-ciphertext input (kernel masquerading): per filter,
    Rescale(x (.) mask_f @ q_l), then the window sums by rotations and adds, then + b_f.
    Output [count*F] (image-major), window (r, c)'s value in slot (r stride) W + c stride."""
    F, kh, kw = K.shape
    l = x.level
    ql = float(ctx.q[l])
    masks = masquerade_masks(K, H, W, stride)
    outs = []
    for f in range(F):
        pt = encode_plain(ctx, masks[f], ql, l)
        pts = np.broadcast_to(pt, (x.count,) + pt.shape)
        y = ctx.rescale(mul_plain(ctx, x, pts, ql))
        for rr in window_rotations(kh, kw, W):
            y = ctx.add(y, rotate(ctx, y, rr, gkeys))
        if bias is not None:
            y = ctx.add_scalar(y, [bias[f]] * y.count)
        outs.append(y)
    data = np.stack([o.data for o in outs], axis=1).reshape((x.count * F,) + outs[0].data.shape[1:])
    return CtArray(data, outs[0].level, outs[0].scale, x.key_id)


# ---------------------------------------------------------------------------------------
# Hoisted tap-by-tap cross-correlation and the class-packed dense layer (NEXT f1 twins of
# the GPU path's masquerade.masked_cc_hoisted / masked_dense_packed).
# Paper: "kernel masquerading ... merging of weights and a respective zeros mask"
# (PAPER.md:279), sums by "key rotation", the dense layer "summed across
# the first axis".  Written from those passages and DESIGN.md §8b; every step
# is an oracle primitive (rotate / rotate_hoisted / mul_plain / add / rescale / add_scalar).

def add_plain(ctx: Context, ct: CtArray, pt_hat: np.ndarray) -> CtArray:
    """ct + plaintext vector: c0 += pt (NTT domain), pt_hat [L'+1][N], L' >= ct.level."""
    out = ct.data.copy()
    for c in range(ct.count):
        for i in range(ct.level + 1):
            out[c, 0, i] = ring.add(ct.data[c, 0, i], pt_hat[i], ctx.q[i])
    return CtArray(out, ct.level, ct.scale, ct.key_id)


def anchor_slots(H: int, W: int, kh: int, kw: int, stride: int):
    """Slot of window (r, c)'s top-left pixel (pixel p in slot p)."""
    Ho, Wo = (H - kh) // stride + 1, (W - kw) // stride + 1
    return [r * stride * W + c * stride for r in range(Ho) for c in range(Wo)]


def masked_cc_hoisted(ctx: Context, x: CtArray, K: np.ndarray, H: int, W: int, stride: int, bias, gkeys,
                      encode) -> CtArray:
    """y_f = Rescale(sum_{u,v} rot(x, u W + v) (.) pt_{f,u,v}) + b_f, pt_{f,u,v} holding
    K_f[u][v] at every window anchor (zeros elsewhere): the tap (u, v) of every window is
    rotated onto the window's anchor, so window (r, c)'s value lands in its anchor slot.
    Rotations share one modulus raise (rotate_hoisted); tap (0, 0) is x itself.
    Output [count*F] image-major.  encode(z, scale) -> int64 poly."""
    F, kh, kw = K.shape
    l = x.level
    ql = float(ctx.q[l])
    n_slots = ctx.n // 2
    anchors = anchor_slots(H, W, kh, kw, stride)
    taps = [(u, v) for u in range(kh) for v in range(kw)]
    rs = [u * W + v for (u, v) in taps]
    rot = {0: x}
    hoisted = rotate_hoisted(ctx, x, [r for r in rs if r != 0], gkeys)
    for r, y in zip([r for r in rs if r != 0], hoisted):
        rot[r] = y
    idx = list(range(l + 1))
    out = np.zeros((x.count * F, 2, l + 1, ctx.n), dtype=np.uint64)
    for f in range(F):
        acc = None
        for (u, v), r in zip(taps, rs):
            z = np.zeros(n_slots)
            z[anchors] = K[f, u, v]
            pt = ctx.signed_to_ntt(np.asarray(encode(z, ql), dtype=np.int64), idx)
            y = mul_plain(ctx, rot[r], np.broadcast_to(pt, (x.count,) + pt.shape), ql)
            acc = y if acc is None else ctx.add(acc, y)
        out[f::F] = acc.data
    y = ctx.rescale(CtArray(out, l, x.scale * ql, x.key_id))
    if bias is not None:
        y = ctx.add_scalar(y, [float(bias[f]) for _ in range(x.count) for f in range(F)])
    return y


def masked_dense_packed(ctx: Context, feats: CtArray, F: int, anchors, Wt: np.ndarray, b, span: int, fill, gkeys,
                        encode) -> CtArray:
    """Class-packed dense: blocks of blk = 2^ceil(log2 span) slots, nb = n_slots / blk
    classes per product ciphertext, G = ceil(O / nb) of them per image.
      1. feature f (slots outside the data region hold the constant fill[f]): subtract
         fill[f] (constant add), then replicate block 0 into every block: r += rot(r, -s)
         for s = blk, 2 blk, ... < n_slots (left rotation by n_slots - s);
      2. product g: sum_f rep_f (.) pt_{g,f}, pt_{g,f}[k blk + anchors[w]] = W[g nb + k][f A + w];
         rescale; block sums r += rot(r, s) for s = 1, 2, ... < blk;
      3. bias: + pt_b with pt_b[k blk] = b_o + sum_f fill[f] sum_w W[o][f A + w] (o = g nb + k),
         encoded at the accumulator's scale.
    Logit o of image i sits in slot (o % nb) blk of ciphertext i G + o // nb."""
    O = Wt.shape[0]
    nimg = feats.count // F
    l = feats.level
    n_slots = ctx.n // 2
    blk = 1
    while blk < span:
        blk *= 2
    nb = n_slots // blk
    G = (O + nb - 1) // nb
    A = len(anchors)
    ql = float(ctx.q[l])
    idx = list(range(l + 1))
    reps = []
    for f in range(F):
        r = feats.select(slice(f, None, F))
        if fill is not None and fill[f] != 0.0:
            r = ctx.add_scalar(r, [-float(fill[f])] * nimg)
        s = blk
        while s < n_slots:
            r = ctx.add(r, rotate(ctx, r, n_slots - s, gkeys))
            s *= 2
        reps.append(r)
    outs = []
    for g in range(G):
        acc = None
        for f in range(F):
            z = np.zeros(n_slots)
            for k in range(nb):
                o = g * nb + k
                if o < O:
                    for w in range(A):
                        z[k * blk + anchors[w]] = Wt[o, f * A + w]
            pt = ctx.signed_to_ntt(np.asarray(encode(z, ql), dtype=np.int64), idx)
            y = mul_plain(ctx, reps[f], np.broadcast_to(pt, (nimg,) + pt.shape), ql)
            acc = y if acc is None else ctx.add(acc, y)
        acc = ctx.rescale(acc)
        s = 1
        while s < blk:
            acc = ctx.add(acc, rotate(ctx, acc, s, gkeys))
            s *= 2
        if b is not None or fill is not None:
            zb = np.zeros(n_slots)
            for k in range(nb):
                o = g * nb + k
                if o < O:
                    v = 0.0 if b is None else float(b[o])
                    if fill is not None:
                        v += sum(float(fill[f]) * float(np.sum(Wt[o, f * A:(f + 1) * A])) for f in range(F))
                    zb[k * blk] = v
            ptb = ctx.signed_to_ntt(np.asarray(encode(zb, acc.scale), dtype=np.int64), list(range(acc.level + 1)))
            acc = add_plain(ctx, acc, ptb)
        outs.append(acc)
    data = np.stack([o.data for o in outs], axis=1).reshape((nimg * G,) + outs[0].data.shape[1:])
    return CtArray(data, outs[0].level, outs[0].scale, feats.key_id)


def packed_logits(ctx: Context, out: CtArray, O: int, span: int) -> np.ndarray:
    """Decrypt masked_dense_packed outputs into [images][O] logits."""
    n_slots = ctx.n // 2
    blk = 1
    while blk < span:
        blk *= 2
    nb = n_slots // blk
    G = (O + nb - 1) // nb
    z = ctx.decrypt(out, n_slots).reshape(out.count // G, G, n_slots)
    return np.stack([z[:, o // nb, (o % nb) * blk] for o in range(O)], axis=1)


def masked_cnn_packed(ctx: Context, x: CtArray, K, kb, Wt, b, H: int, W: int, stride: int, coeffs, gkeys,
                      encode) -> CtArray:
    """The paper-layout CNN: hoisted masked CC -> sigma -> class-packed dense, with the CC
    bias' activation sigma(kb_f) (present in every slot outside the data region)
    compensated inside the dense layer."""
    from .layers import poly_activation
    K = np.asarray(K, dtype=np.float64)
    F, kh, kw = K.shape
    cc = masked_cc_hoisted(ctx, x, K, H, W, stride, kb, gkeys, encode)
    act = poly_activation(ctx, cc, coeffs)
    kbv = np.zeros(F) if kb is None else np.asarray(kb, dtype=np.float64)
    fill = [float(sum(c * v ** k for k, c in enumerate(coeffs))) for v in kbv]
    return masked_dense_packed(ctx, act, F, anchor_slots(H, W, kh, kw, stride), np.asarray(Wt, dtype=np.float64), b,
                               H * W, fill, gkeys, encode)
