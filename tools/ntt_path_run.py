"""Driver for ncu captures of the plain batched NTT on one arithmetic path:
python tools/ntt_path_run.py fp40|int60 fwd|inv  (runs the transform 3 times)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2110_13638_b200 import edl

path, d = sys.argv[1], sys.argv[2]
bits = [60] * 6 if path == "int60" else [40] * 5 + [60]
ctx = edl.Context(edl.params_from_bits(14, bits))
lvl = len(bits) - 2
polys = 512
t = torch.randint(0, 2 ** 39, (polys * (lvl + 1) << 14,), dtype=torch.int64, device="cuda")
for _ in range(3):
    ctx.ntt_(t, polys, lvl, d == "inv")
torch.cuda.synchronize()
print("ok")
