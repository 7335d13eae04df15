import sys, json
sys.path.insert(0, '/root/repo')
import torch
from paper_2110_13638_b200 import edl
for logn, L in ((14, 6), (14, 12), (14, 24)):
    bits = [60] + [40] * (L - 2) + [60] + [60]
    ctx = edl.Context(edl.params_from_bits(logn, bits)).keygen(3)
    lvl = L - 1
    x = ctx.empty(256, lvl); y = ctx.empty(256, lvl)
    g = torch.Generator(device="cuda").manual_seed(3)
    for t in (x.tensor, y.tensor):
        t.copy_(torch.randint(0, 2 ** 39, (t.numel(),), dtype=torch.int64, device="cuda", generator=g))
    x.scale = y.scale = 2.0 ** 40; x.key_id = y.key_id = ctx.key_id
    ctx.mul_relin(x, y); torch.cuda.synchronize()
    ctx.profile(True); ctx.mul_relin(x, y); p = ctx.profile_read(); ctx.profile(False)
    print(logn, L, {k: round(v[0], 3) for k, v in p.items()})
    ctx.close(); torch.cuda.empty_cache()
