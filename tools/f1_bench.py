"""NEXT f1 measurement: C1's CNN in the paper's own layout (one Fashion-MNIST-shaped image
per ciphertext, kernel masquerading, Galois-rotation window and class sums) on B images;
device-timed images/s and the max |decrypted - float64| logit error (numpy reference).

Usage: python tools/f1_bench.py [--images 64] [--reps 3]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2110_13638_b200 import edl, masquerade
from synth import c1_images, c1_weights


def float64_logits(imgs, K, kb, W, b):
    B = imgs.shape[0]
    cc = np.zeros((B, 5, 7, 7))
    for f in range(5):
        for r in range(7):
            for c in range(7):
                cc[:, f, r, c] = np.sum(imgs[:, 4 * r:4 * r + 4, 4 * c:4 * c + 4] * K[f], axis=(1, 2)) + kb[f]
    a = 0.5 + 0.197 * cc - 0.004 * cc ** 3
    return a.reshape(B, 245) @ W.T + b


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--images", type=int, default=64)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    ctx = edl.Context(edl.params_from_depth(4)).keygen(1)
    rots = masquerade.network_rotations(28, 28, 4, 4)
    ctx.galois_keygen(7, rots)
    K, kb, W, b = c1_weights()
    imgs = c1_images(a.images, 2110)
    x = ctx.encrypt(imgs.reshape(a.images, 784), enc_seed=2)
    out = masquerade.masked_cnn(ctx, x, K, kb, W, b)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(ctx.stream)
    for _ in range(a.reps):
        out = masquerade.masked_cnn(ctx, x, K, kb, W, b)
    e1.record(ctx.stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.reps
    got = ctx.decrypt(out, 1)[:, 0].reshape(a.images, 10)
    err = float(np.max(np.abs(got - float64_logits(imgs, K, kb, W, b))))
    # class-packed dense: replicate features into 1024-slot blocks, one product per feature,
    # in-block sums (35 dense rotations per image instead of 100)
    ctx.galois_keygen(8, masquerade.packed_rotations(ctx.n // 2, 784))
    outp = masquerade.masked_cnn(ctx, x, K, kb, W, b, packed=True)
    torch.cuda.synchronize()
    e0.record(ctx.stream)
    for _ in range(a.reps):
        outp = masquerade.masked_cnn(ctx, x, K, kb, W, b, packed=True)
    e1.record(ctx.stream)
    torch.cuda.synchronize()
    msp = e0.elapsed_time(e1) / a.reps
    errp = float(np.max(np.abs(masquerade.packed_logits(ctx, outp, 10, 784) - float64_logits(imgs, K, kb, W, b))))
    # + CC from hoisted tap rotations (15 rotations sharing one modulus raise per image)
    ctx.galois_keygen(9, [r for r in masquerade.tap_rotations(4, 4, 28) if r])
    outh = masquerade.masked_cnn(ctx, x, K, kb, W, b, packed=True, hoisted=True)
    torch.cuda.synchronize()
    e0.record(ctx.stream)
    for _ in range(a.reps):
        outh = masquerade.masked_cnn(ctx, x, K, kb, W, b, packed=True, hoisted=True)
    e1.record(ctx.stream)
    torch.cuda.synchronize()
    msh = e0.elapsed_time(e1) / a.reps
    errh = float(np.max(np.abs(masquerade.packed_logits(ctx, outh, 10, 784) - float64_logits(imgs, K, kb, W, b))))
    print(json.dumps({"config": "C1 CNN in the paper's layout: one 28x28 image per ciphertext (N=2^14), masked CC "
                                "5x4x4/4 + 4 rotations/filter, sigma_a, masked dense with 10 rotations/class",
                      "images": a.images, "rotations_per_image": 5 * 4 + 10 * len(masquerade.sum_rotations(784)),
                      "galois_keys": len(rots), "ms_per_batch": ms, "images_per_s": a.images / (ms / 1e3),
                      "max_abs_err_vs_float64": err,
                      "packed_dense": {"rotations_per_image": 5 * 4 + 5 * 3 + 2 * 10, "ms_per_batch": msp,
                                       "images_per_s": a.images / (msp / 1e3), "max_abs_err_vs_float64": errp},
                      "packed_dense_hoisted_cc": {"rotations_per_image": 15 + 5 * 3 + 2 * 10,
                                                  "note": "15 CC rotations hoisted (one modulus raise per image)",
                                                  "ms_per_batch": msh, "images_per_s": a.images / (msh / 1e3),
                                                  "max_abs_err_vs_float64": errh}}))


if __name__ == "__main__":
    main()
