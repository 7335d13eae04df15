"""NEXT-row measurements at C1 scale, device-timed on the library's stream:

f2 activations over the 245 CC-output ciphertexts of a C1 batch (level 3 -> level 1/2):
   sigma_a (degree 3, the hot path's), ReLU_a (degree 2), x^2 (C0's) and
   the linear sigma, ciphertexts/s;
f3 client path for one 8192-image C1 batch: GPU encode (784 pixel vectors -> polys) +
   public-key encrypt, secret-key encrypt, and device decrypt + decode of the 10 logit
   ciphertexts, ciphertexts/s and images/s.

Usage: python tools/f23_bench.py [--reps 5]
(Coefficients of ReLU_a are restated here from PAPER.md:416, the library takes any degree-2
schedule; no oracle is imported.)
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2110_13638_b200 import edl
from paper_2110_13638_b200.networks import SIGMA_A
from synth import c1_images, c1_slots


def timed(stream, fn, reps):
    fn()
    stream.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(reps):
        fn()
    b.record(stream)
    stream.synchronize()
    return a.elapsed_time(b) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = edl.Context(edl.params_from_depth(4), stream=stream).keygen(1)
    res = {}
    # f2: activations on 245 ciphertexts at level 3 (the CC outputs' level)
    g = torch.Generator(device="cuda").manual_seed(5)
    x = ctx.empty(245, 3)
    x.tensor.copy_(torch.randint(0, 2 ** 39, (x.tensor.numel(),), dtype=torch.int64, device="cuda", generator=g))
    x.scale, x.key_id = 2.0 ** 40, ctx.key_id
    relu_a = (1.0 / (3.0 * np.pi), 0.5, 4.0 / (3.0 * np.pi))   # R_a(x), q = 1
    for name, cf in (("sigma_a", SIGMA_A), ("relu_a", relu_a), ("square", (0.0, 0.0, 1.0)), ("sigma_linear", (0.5, 0.197))):
        ms = timed(stream, lambda: ctx.poly_activation(x, cf), a.reps)
        res[f"f2_{name}_cts_per_s"] = 245 / ms * 1e3
        res[f"f2_{name}_ms_per_245_cts"] = ms
    # f3: client path for one C1 batch
    slots = torch.from_numpy(c1_slots(c1_images(8192, 2110))).cuda()          # [784][8192]
    ms_enc = timed(stream, lambda: ctx.encode_device(slots), a.reps)
    polys = ctx.encode_device(slots)
    ms_pk = timed(stream, lambda: ctx.encrypt_poly(polys, scale=2.0 ** 40, enc_seed=2), a.reps)
    ms_sk = timed(stream, lambda: ctx.encrypt_poly_sk(polys, scale=2.0 ** 40, enc_seed=3), a.reps)
    out = ctx.empty(10, 0)
    out.tensor.copy_(torch.randint(0, 2 ** 39, (out.tensor.numel(),), dtype=torch.int64, device="cuda", generator=g))
    out.scale, out.key_id = 2.0 ** 40, ctx.key_id
    ms_dec = timed(stream, lambda: ctx.decrypt_device(out, 8192), a.reps)
    res.update({"f3_encode_784x8192_ms": ms_enc, "f3_encrypt_pk_784_ms": ms_pk, "f3_encrypt_sk_784_ms": ms_sk,
                "f3_decrypt_decode_10_ms": ms_dec,
                "f3_client_images_per_s_pk": 8192 / ((ms_enc + ms_pk + ms_dec) / 1e3),
                "f3_client_images_per_s_sk": 8192 / ((ms_enc + ms_sk + ms_dec) / 1e3)})
    print(json.dumps({k: (round(v, 4) if isinstance(v, float) else v) for k, v in res.items()}))


if __name__ == "__main__":
    main()
