"""Per-arithmetic-path NTT rates: the batched plain NTT/INTT (k_ntt_limbs) over chains whose
primes are all 60-bit (integer Shoup butterflies) or all 40-bit (FP64-pipe butterflies) at
N = 2^14, against each path's register-only butterfly ceiling (edl_bfly_peak).  Shows which
path loses the most to memory / exchange / pass overheads.  `EDL_LIB` selects a build."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2110_13638_b200 import edl
from tools.ntt_bench import time_ms


def main():
    res = {"lib": os.environ.get("EDL_LIB", "default")}
    logn = 14
    n = 1 << logn
    bfly = (n // 2) * logn
    for name, bits in (("int60", [60] * 6), ("fp40", [40] * 5 + [60])):
        ctx = edl.Context(edl.params_from_bits(logn, bits))
        lvl = len(bits) - 2
        polys = 512
        t = torch.randint(0, 2 ** 39, (polys * (lvl + 1) * n,), dtype=torch.int64, device="cuda")
        limbs = polys * (lvl + 1)
        f = time_ms(lambda: ctx.ntt_(t, polys, lvl, False))
        i = time_ms(lambda: ctx.ntt_(t, polys, lvl, True))
        pk = ctx.bfly_peak(0) / 1e9
        res[name] = {"fwd_Mlimb_s": round(limbs / f / 1e3, 3), "inv_Mlimb_s": round(limbs / i / 1e3, 3),
                     "fwd_Gbfly_s": round(limbs * bfly / f / 1e6, 1), "inv_Gbfly_s": round(limbs * bfly / i / 1e6, 1),
                     "peak_Gbfly_s": round(pk, 1), "fwd_frac": round(limbs * bfly / f / 1e6 / pk, 3),
                     "inv_frac": round(limbs * bfly / i / 1e6 / pk, 3)}
        del t, ctx
    print(json.dumps(res))


if __name__ == "__main__":
    main()
