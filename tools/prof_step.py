"""Profiling driver for ncu: one plain forward + inverse NTT batch at N=2^14 (C1 chain),
then one C1 step (CC -> sigma_a -> dense).  Keygen/encrypt kernels run first; capture
the hot kernels with  ncu -k regex:'^k_(ntt|cc|rescale|relin|dense|add)' ...
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2110_13638_b200 import edl
from paper_2110_13638_b200.networks import C1Net
from synth import c1_weights


def main():
    ctx = edl.Context(edl.params_from_depth(4)).keygen(1)
    K, kb, W, b = c1_weights()
    polys = torch.randint(-2 ** 39, 2 ** 39, (784, 1 << 14), dtype=torch.int64, device="cuda")
    x = ctx.encrypt_poly(polys, scale=2.0 ** 40, enc_seed=2)
    net = C1Net(ctx, K, kb, W, b)
    torch.cuda.synchronize()
    if "--step-only" not in sys.argv:
        t = torch.randint(0, 2 ** 39, (256 * 5 * (1 << 14),), dtype=torch.int64, device="cuda")
        ctx.ntt_(t, 256, 4, False)
        ctx.ntt_(t, 256, 4, True)
    torch.cuda.synchronize()
    net.forward(x)
    torch.cuda.synchronize()
    print("prof_step ok")


if __name__ == "__main__":
    main()
