"""Microbench: batched NTT/INTT limb-transforms/s through edl_ntt (C2-style), plus the
C1 step time.  `EDL_LIB=<path> python tools/ntt_bench.py` compares library variants."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2110_13638_b200 import edl


def time_ms(fn, reps=5):
    st = torch.cuda.current_stream()
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(reps):
        fn()
    b.record(st)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    res = {"lib": os.environ.get("EDL_LIB", "default")}
    for logn, bits in ((13, [60, 40, 40, 60]), (14, [60, 40, 40, 40, 40, 60])):
        try:
            ctx = edl.Context(edl.params_from_bits(logn, bits))
        except edl.EdlError:
            continue   # ring degree not compiled into this (trimmed) library
        lvl = len(bits) - 2
        polys = 1024 if logn == 14 else 2048
        n = 1 << logn
        t = torch.randint(0, 2 ** 39, (polys * (lvl + 1) * n,), dtype=torch.int64, device="cuda")
        f = time_ms(lambda: ctx.ntt_(t, polys, lvl, False))
        i = time_ms(lambda: ctx.ntt_(t, polys, lvl, True))
        limbs = polys * (lvl + 1)
        res[f"fwd_2^{logn}_Mlimb_per_s"] = limbs / f / 1e3
        res[f"inv_2^{logn}_Mlimb_per_s"] = limbs / i / 1e3
        res[f"fwd_2^{logn}_GBps"] = limbs * 16 * n / f / 1e6
    from paper_2110_13638_b200.networks import C1Net
    from synth import c1_weights
    ctx = edl.Context(edl.params_from_depth(4)).keygen(1)
    K, kb, W, b = c1_weights()
    polys = torch.randint(-2 ** 39, 2 ** 39, (784, 1 << 14), dtype=torch.int64, device="cuda")
    x = ctx.encrypt_poly(polys, scale=2.0 ** 40, enc_seed=2)
    net = C1Net(ctx, K, kb, W, b)
    res["c1_step_ms"] = time_ms(lambda: net.forward(x), reps=3)
    for ev in os.environ.get("EDL_BENCH_ENVS", "").split(";"):
        if ev:   # the same C1 step under a context-creation switch, e.g. EDL_RAISE_FUSED=1
            k_, v_ = ev.split("=")
            os.environ[k_] = v_
            cx = edl.Context(edl.params_from_depth(4)).keygen(1)
            xc = cx.encrypt_poly(polys, scale=2.0 ** 40, enc_seed=2)
            nc = C1Net(cx, K, kb, W, b)
            res[f"c1_step_ms[{ev}]"] = time_ms(lambda: nc.forward(xc), reps=3)
            cx.profile(True)
            nc.forward(xc)
            res[f"c1_kernels_ms[{ev}]"] = {k: round(v[0], 3) for k, v in cx.profile_read().items()}
            cx.profile(False)
            del nc, xc, cx
            os.environ.pop(k_)
    for ch in os.environ.get("EDL_BENCH_CHUNKS", "").split(","):
        if ch:   # the same C1 step with key switches in chunks (EDL_KS_CHUNK, read at context creation)
            os.environ["EDL_KS_CHUNK"] = ch
            cx = edl.Context(edl.params_from_depth(4)).keygen(1)
            xc = cx.encrypt_poly(polys, scale=2.0 ** 40, enc_seed=2)
            nc = C1Net(cx, K, kb, W, b)
            res[f"c1_step_ms_chunk{ch}"] = time_ms(lambda: nc.forward(xc), reps=3)
            del nc, xc, cx
            os.environ.pop("EDL_KS_CHUNK")
    ctx.profile(True)
    net.forward(x)
    res["c1_kernels_ms"] = {k: round(v[0], 3) for k, v in ctx.profile_read().items()}
    ctx.profile(False)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
