"""C2 RNS kernel microbenchmark (BASELINE.json configs[2]).

Sweep N in {2^13, 2^14, 2^15, 2^16} x data limbs L in {3, 6, 12, 24} (chain [60] + [40]*(L-2)
+ [60] data primes plus one 60-bit special prime) on a batch of 256 ciphertexts
of Philox/uniform random residues, and report per point:
  * NTT and INTT limb-transforms/s (256 * 2 * L limbs per call),
  * pointwise modmul GB/s (ct x scalar, 24 B per element: read + write + constant),
  * key-switches/s (tensor + relinearisation at level L-1, 256 per call),
  * rescales/s (level L-1 -> L-2, 256 per call),
all device-timed with CUDA events on the library's stream (median of reps after warm-up).

Usage: python tools/c2_bench.py [--logn 13 14 15 16] [--limbs 3 6 12 24] [--batch 256]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2110_13638_b200 import edl


def chain(L):
    return [60] + [40] * (L - 2) + [60] + [60]


def timed(ctx, fn, reps):
    st = ctx.stream
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        fn()
        b.record(st)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def point(logn, L, batch, reps):
    n = 1 << logn
    ctx = edl.Context(edl.params_from_bits(logn, chain(L))).keygen(3)
    lvl = L - 1
    words = batch * 2 * L * n
    x = ctx.empty(batch, lvl)
    y = ctx.empty(batch, lvl)
    g = torch.Generator(device="cuda").manual_seed(3)
    for t in (x.tensor, y.tensor):
        # residues below the smallest prime of the chain (uniform in [0, 2^39))
        t.copy_(torch.randint(0, 2 ** 39, (t.numel(),), dtype=torch.int64, device="cuda", generator=g))
    x.scale = y.scale = 2.0 ** 40
    x.key_id = y.key_id = ctx.key_id
    res = {"logn": logn, "limbs": L, "batch": batch}
    ms = timed(ctx, lambda: ctx.ntt_(x.tensor, batch * 2, lvl, False), reps)
    res["ntt_Mlimb_per_s"] = batch * 2 * L / ms / 1e3
    ms = timed(ctx, lambda: ctx.ntt_(x.tensor, batch * 2, lvl, True), reps)
    res["intt_Mlimb_per_s"] = batch * 2 * L / ms / 1e3
    w = np.full(batch, 0.37)
    ms = timed(ctx, lambda: ctx.pt_mul(x, w, 2.0 ** 20), reps)
    res["modmul_GBps"] = words * 16 / ms / 1e6
    ms = timed(ctx, lambda: ctx.mul_relin(x, y), max(2, reps // 2))
    res["keyswitch_per_s"] = batch / ms * 1e3
    ms = timed(ctx, lambda: ctx.rescale(x), reps)
    res["rescale_per_s"] = batch / ms * 1e3
    ctx.close()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--logn", type=int, nargs="+", default=[13, 14, 15, 16])
    ap.add_argument("--limbs", type=int, nargs="+", default=[3, 6, 12, 24])
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    for logn in a.logn:
        for L in a.limbs:
            r = point(logn, L, a.batch, a.reps)
            print(json.dumps({k: (round(v, 3) if isinstance(v, float) else v) for k, v in r.items()}), flush=True)
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
