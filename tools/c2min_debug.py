import sys, os
sys.path.insert(0, '/root/repo')
import torch
from paper_2110_13638_b200 import edl
logn, L = int(sys.argv[1]), int(sys.argv[2])
bits = [60] + [40] * (L - 2) + [60] + [60]
ctx = edl.Context(edl.params_from_bits(logn, bits)).keygen(3)
lvl = L - 1
batch = int(sys.argv[3]) if len(sys.argv) > 3 else 4
x = ctx.empty(batch, lvl); y = ctx.empty(batch, lvl)
g = torch.Generator(device="cuda").manual_seed(3)
for t in (x.tensor, y.tensor):
    t.copy_(torch.randint(0, 2 ** 39, (t.numel(),), dtype=torch.int64, device="cuda", generator=g))
x.scale = y.scale = 2.0 ** 40
x.key_id = y.key_id = ctx.key_id
ctx.profile(True)
for step in ("ntt", "relin", "rescale"):
    if step == "ntt": ctx.ntt_(x.tensor, batch * 2, lvl, False)
    if step == "relin": z = ctx.mul_relin(x, y)
    if step == "rescale": ctx.rescale(x)
    torch.cuda.synchronize()
    print(step, "ok", flush=True)
