"""ncu driver: one batched forward + inverse NTT at N=2^14 (C1 chain, 256 polys)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2110_13638_b200 import edl

ctx = edl.Context(edl.params_from_bits(14, [60, 40, 40, 40, 40, 60]))
t = torch.randint(0, 2 ** 39, (512 * 5 * (1 << 14),), dtype=torch.int64, device="cuda")
for _ in range(2):
    ctx.ntt_(t, 512, 4, False)
    ctx.ntt_(t, 512, 4, True)
torch.cuda.synchronize()
print("prof_ntt ok")
