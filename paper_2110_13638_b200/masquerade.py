"""The paper's own CNN layout (NEXT f1): one image per ciphertext, kernel masquerading
(SPEC.md `masquerade_kernel` / `cc_forward`).

"Kernel-masquerading shall mean the merging of weights and a respective zeros mask into a
sparse n-dimensional array such that they become a single operation conducted on the
input cyphertext".  With non-overlapping windows (C1: 4x4, stride 4) one
mask per filter carries the filter at every window position, so a single plaintext
product covers all windows of that filter; the products of a window are then summed into
its top-left slot by log2(kh) + log2(kw) rotations and additions (the paper's "key
rotation to sum", done here with Galois rotations on the GPU instead of a client round
trip).  Every step is a C-ABI call (plaintext-vector product, rescale, rotate, add).
"""
from __future__ import annotations

from typing import Callable, List, Optional, Sequence

import numpy as np

from .edl import Context, CtArray


def masquerade_masks(K: np.ndarray, H: int, W: int, stride: int) -> np.ndarray:
    """[F][H*W]: filter f's weights at every window position (zeros elsewhere)."""
    F, kh, kw = K.shape
    if kh > H or kw > W:
        raise ValueError("kernel larger than input")
    Ho, Wo = (H - kh) // stride + 1, (W - kw) // stride + 1
    masks = np.zeros((F, H * W))
    for r in range(Ho):
        for c in range(Wo):
            for u in range(kh):
                base = (r * stride + u) * W + c * stride
                masks[:, base:base + kw] += K[:, u, :]
    return masks


def window_rotations(kh: int, kw: int, W: int) -> List[int]:
    """Rotations summing a kh x kw window (power-of-two sides) into its top-left slot."""
    if kh & (kh - 1) or kw & (kw - 1):
        raise ValueError("window sums by rotation need power-of-two kernel sides")
    out, s = [], 1
    while s < kw:
        out.append(s)
        s *= 2
    s = 1
    while s < kh:
        out.append(s * W)
        s *= 2
    return out


def anchor_slots(H: int, W: int, kh: int, kw: int, stride: int) -> List[int]:
    Ho, Wo = (H - kh) // stride + 1, (W - kw) // stride + 1
    return [(r * stride) * W + c * stride for r in range(Ho) for c in range(Wo)]


def masked_cc(ctx: Context, x: CtArray, K: np.ndarray, H: int, W: int, stride: int,
              bias: Optional[Sequence[float]] = None, encode: Optional[Callable] = None) -> CtArray:
    """x: one image per ciphertext (pixel p in slot p).  Returns [count*F] ciphertexts
    (image-major) whose window (r, c) value sits in slot anchor_slots(...)[r*Wo + c];
    level x.level - 1, scale x.scale.  Needs Galois keys for window_rotations(kh, kw, W).
    `encode(z, scale) -> int64 poly` picks the slot encoder (default: the library's host
    FFT); the masks then enter through edl_encode_pt_poly."""
    F, kh, kw = K.shape
    l = x.level
    ql = float(ctx.params.qs[l])
    masks = masquerade_masks(np.asarray(K, dtype=np.float64), H, W, stride)
    outs = []
    for f in range(F):
        poly = ctx.encode(masks[f][None, :], ql) if encode is None else np.asarray(encode(masks[f], ql))[None, :]
        pt = ctx.encode_pt_poly(poly, l)
        y = ctx.rescale(ctx.pt_vec_mul(x, pt, 1, l, ql))
        for r in window_rotations(kh, kw, W):
            y = ctx.add(y, ctx.rotate(y, r))
        if bias is not None:
            y = ctx.pt_add(y, [float(bias[f])] * y.count)
        outs.append(y)
    torch = ctx.torch
    t = torch.stack([o.tensor.view(x.count, -1) for o in outs], dim=1).reshape(-1)
    return CtArray(t, x.count * F, outs[0].level, outs[0].scale, outs[0].key_id)


def tap_rotations(kh: int, kw: int, W: int) -> List[int]:
    """Rotations bringing tap (u, v) of every window onto the window's anchor: u W + v."""
    return [u * W + v for u in range(kh) for v in range(kw)]


def masked_cc_hoisted(ctx: Context, x: CtArray, K: np.ndarray, H: int, W: int, stride: int,
                      bias: Optional[Sequence[float]] = None, encode: Optional[Callable] = None) -> CtArray:
    """The masked CC computed tap by tap from hoisted rotations of the input (one modulus
    raise for all kh*kw - 1 rotations, `edl_rotate_hoisted`):
        y_f = sum_{u,v} rot(x, u W + v) (.) pt_{f,u,v},   pt_{f,u,v}[anchor] = K_f[u][v],
    so every window's value lands on its anchor slot and every other slot holds 0 (+ the
    bias).  Same output layout, level and scale as `masked_cc`; the 5 x 16 plaintexts are
    encoded on the GPU (f3) in one batch, or by `encode(z, scale) -> int64 poly` when given.
    Needs Galois keys for tap_rotations(kh, kw, W)."""
    F, kh, kw = K.shape
    l = x.level
    ql = float(ctx.params.qs[l])
    n_slots = ctx.n // 2
    anchors = np.asarray(anchor_slots(H, W, kh, kw, stride))
    taps = tap_rotations(kh, kw, W)
    z = np.zeros((F * len(taps), n_slots))
    for f in range(F):
        for k, (u, v) in enumerate((u, v) for u in range(kh) for v in range(kw)):
            z[f * len(taps) + k, anchors] = K[f, u, v]
    T = len(taps)
    polys = ctx.encode_device(z, ql) if encode is None else np.stack([np.asarray(encode(v, ql)) for v in z])
    pts = ctx.encode_pt_poly(polys, l)                              # [F][T][l+1][N]
    words = x.tensor.numel()
    big = ctx.torch.empty(T * words, dtype=ctx.torch.int64, device=x.tensor.device)
    views = [CtArray(big[k * words:(k + 1) * words], x.count, l, x.scale, x.key_id) for k in range(T)]
    ctx.rotate_hoisted(x, taps, outs=views)     # taps[0] = 0: a copy of x
    rots = CtArray(big, T * x.count, l, x.scale, x.key_id)
    y = ctx.rescale(ctx.pt_mac_multi(rots, T, pts, F, l, ql))   # [count*F], image-major
    if bias is not None:
        y = ctx.pt_add(y, [float(bias[f]) for _ in range(x.count) for f in range(F)])
    return y


def sum_rotations(span: int) -> List[int]:
    """Rotations 1, 2, 4, ... summing slots [0, span) (zero elsewhere) into slot 0."""
    out, s = [], 1
    while s < span:
        out.append(s)
        s *= 2
    return out


def network_rotations(H: int, W: int, kh: int, kw: int) -> List[int]:
    return sorted(set(window_rotations(kh, kw, W) + sum_rotations(H * W)))


def masked_dense(ctx: Context, feats: CtArray, F: int, anchors: Sequence[int], Wt: np.ndarray, b, span: int,
                 encode: Optional[Callable] = None) -> CtArray:
    """Dense layer on the masked-CC feature ciphertexts [count*F] (image-major, window w's
    feature in slot anchors[w]): class o = sum_f Rescale(feat_f (.) pt_{o,f}) with
    pt_{o,f}[anchors[w]] = W[o][f*len(anchors) + w], summed over all slots by rotations
    into slot 0, + b_o.  Returns [count*O] (image-major), logit o of an image in slot 0."""
    O = Wt.shape[0]
    nimg = feats.count // F
    l = feats.level
    ql = float(ctx.params.qs[l])
    words = 2 * (l + 1) * ctx.n
    fv = feats.tensor.view(nimg, F, words)
    torch = ctx.torch
    outs = []
    for o in range(O):
        acc = None
        for f in range(F):
            z = np.zeros(span)
            z[list(anchors)] = Wt[o, f * len(anchors):(f + 1) * len(anchors)]
            poly = ctx.encode(z[None, :], ql) if encode is None else np.asarray(encode(z, ql))[None, :]
            pt = ctx.encode_pt_poly(poly, l)
            xf = CtArray(fv[:, f].contiguous().view(-1), nimg, l, feats.scale, feats.key_id)
            y = ctx.pt_vec_mul(xf, pt, 1, l, ql)
            acc = y if acc is None else ctx.add(acc, y)
        acc = ctx.rescale(acc)
        for r in sum_rotations(span):
            acc = ctx.add(acc, ctx.rotate(acc, r))
        if b is not None:
            acc = ctx.pt_add(acc, [float(b[o])] * acc.count)
        outs.append(acc)
    t = torch.stack([x.tensor.view(nimg, -1) for x in outs], dim=1).reshape(-1)
    return CtArray(t, nimg * O, outs[0].level, outs[0].scale, outs[0].key_id)


def packed_block(span: int) -> int:
    """Smallest power of two >= span: the slot block one class occupies in the packed dense."""
    blk = 1
    while blk < span:
        blk *= 2
    return blk


def packed_rotations(n_slots: int, span: int) -> List[int]:
    """Rotations of the packed dense: replication of block 0 into every block (right shifts
    by blk, 2 blk, ..., as left rotations n_slots - s) and the in-block sums 1 .. blk/2."""
    blk = packed_block(span)
    reps, s = [], blk
    while s < n_slots:
        reps.append(n_slots - s)
        s *= 2
    return reps + sum_rotations(blk)


def masked_dense_packed(ctx: Context, feats: CtArray, F: int, anchors: Sequence[int], Wt: np.ndarray, b,
                        span: int, fill: Optional[Sequence[float]] = None,
                        encode: Optional[Callable] = None) -> CtArray:
    """Dense layer with the classes packed into slot blocks (fewer rotations than
    `masked_dense`'s 10 per class): every feature ciphertext is replicated into the
    n_slots / blk blocks of blk = 2^ceil(log2 span) slots (log2(n_slots / blk) rotations,
    block 0 holds the features and zeros above span), one plaintext product per feature
    puts class o's weights in block o (o < n_slots / blk; further classes in a second
    product ciphertext over the same replicas), and log2(blk) rotations sum every block
    into its first slot.  Returns [count * G] ciphertexts, G = ceil(O / (n_slots / blk)):
    logit o of image i in slot (o % nb) * blk of ciphertext i * G + o // nb; bias added
    per block through a trivially encrypted plaintext vector.
    Feature f holds the constant fill[f] in every slot outside the masked CC's data region
    (C1: sigma_a(kb_f), the activation of the CC bias that pt_add put in every slot); it is
    subtracted from every slot before the replication (no level used) so the other blocks'
    copies add exact zeros at the anchors, and sum_f fill[f] * sum_w W[o][f*A + w] is added
    back through the bias (a ct + plaintext-vector add, edl_ct_pt_vec_add).  Plaintexts come
    from the library's host encoder, or from `encode(z, scale) -> int64 poly` when given.
    C1: 5 * 3 replication + 2 * 10 block-sum rotations = 35 per image instead of 100."""
    O = Wt.shape[0]
    nimg = feats.count // F
    l = feats.level
    n_slots = ctx.n // 2
    blk = packed_block(span)
    nb = n_slots // blk
    G = (O + nb - 1) // nb
    ql = float(ctx.params.qs[l])
    words = 2 * (l + 1) * ctx.n
    fv = feats.tensor.view(nimg, F, words)
    torch = ctx.torch

    def enc_pt(z, scale, level):
        if encode is None:
            return ctx.encode_pt(z[None, :], scale, level)
        return ctx.encode_pt_poly(np.asarray(encode(z, scale))[None, :], level)

    reps = []
    for f in range(F):
        r = CtArray(fv[:, f].contiguous().view(-1), nimg, l, feats.scale, feats.key_id)
        if fill is not None and fill[f] != 0.0:
            r = ctx.pt_add(r, [-float(fill[f])] * nimg)
        s = blk
        while s < n_slots:
            r = ctx.add(r, ctx.rotate(r, n_slots - s))
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
                    z[k * blk + np.asarray(anchors)] = Wt[o, f * len(anchors):(f + 1) * len(anchors)]
            pt = enc_pt(z, ql, l)
            y = ctx.pt_vec_mul(reps[f], pt, 1, l, ql)
            acc = y if acc is None else ctx.add(acc, y)
        acc = ctx.rescale(acc)
        for r in sum_rotations(blk):
            acc = ctx.add(acc, ctx.rotate(acc, r))
        if b is not None or fill is not None:
            zb = np.zeros(n_slots)
            for k in range(nb):
                o = g * nb + k
                if o < O:
                    zb[k * blk] = 0.0 if b is None else float(b[o])
                    if fill is not None:
                        A = len(anchors)
                        zb[k * blk] += sum(float(fill[f]) * float(np.sum(Wt[o, f * A:(f + 1) * A])) for f in range(F))
            acc = ctx.pt_vec_add(acc, enc_pt(zb, acc.scale, acc.level), 1, acc.level)
        outs.append(acc)
    t = torch.stack([x.tensor.view(nimg, -1) for x in outs], dim=1).reshape(-1)
    return CtArray(t, nimg * G, outs[0].level, outs[0].scale, outs[0].key_id)


def packed_logits(ctx: Context, out: CtArray, O: int, span: int) -> np.ndarray:
    """Decrypt `masked_dense_packed` outputs into [images][O] logits."""
    n_slots = ctx.n // 2
    blk = packed_block(span)
    nb = n_slots // blk
    G = (O + nb - 1) // nb
    z = ctx.decrypt(out, n_slots).reshape(out.count // G, G, n_slots)
    return np.stack([z[:, o // nb, (o % nb) * blk] for o in range(O)], axis=1)


def masked_cnn(ctx: Context, x: CtArray, K, kb, Wt, b, H: int = 28, W: int = 28, stride: int = 4,
               coeffs=(0.5, 0.197, 0.0, -0.004), encode: Optional[Callable] = None,
               packed: bool = False, hoisted: bool = False) -> CtArray:
    """C1's architecture in the paper's layout: masked CC -> sigma_a -> masked dense.
    x: one image per ciphertext (level >= 4).  Returns [count*10] ciphertexts, logit o of
    image i in slot 0 of ciphertext i*10 + o; with packed=True the dense is
    `masked_dense_packed` (read the logits with `packed_logits`); with hoisted=True the CC is
    `masked_cc_hoisted`."""
    F, kh, kw = np.asarray(K).shape
    if hoisted:
        cc = masked_cc_hoisted(ctx, x, np.asarray(K, dtype=np.float64), H, W, stride, kb, encode=encode)
    else:
        cc = masked_cc(ctx, x, K, H, W, stride, kb, encode=encode)
    act = ctx.poly_activation(cc, coeffs)
    if packed:
        kbv = np.zeros(F) if kb is None else np.asarray(kb, dtype=np.float64)
        fill = [float(sum(c * v ** k for k, c in enumerate(coeffs))) for v in kbv]   # sigma(kb_f)
        return masked_dense_packed(ctx, act, F, anchor_slots(H, W, kh, kw, stride), np.asarray(Wt), b, H * W,
                                   fill=fill, encode=encode)
    return masked_dense(ctx, act, F, anchor_slots(H, W, kh, kw, stride), np.asarray(Wt), b, H * W, encode=encode)
