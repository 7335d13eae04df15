"""Probe: C1 throughput with consecutive batches alternating over two contexts (each with its
own stream pair and scratch) against one context, same total number of batches.
Usage: python tools/pipe_probe.py [steps]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2110_13638_b200 import edl
from paper_2110_13638_b200.networks import C1Net
from synth import c1_images, c1_slots, c1_weights


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    K, kb, W, b = c1_weights()
    ctxs, nets, xs, streams = [], [], [], []
    NC = 3
    for i in range(NC):
        st = torch.cuda.Stream()
        ctx = edl.Context(edl.params_from_depth(4), device=0, stream=st).keygen(1)
        with torch.cuda.stream(st):
            polys = torch.from_numpy(ctx.encode(c1_slots(c1_images(8192, 2110 + i)))).to("cuda:0")
            x = ctx.encrypt_poly(polys, scale=float(2 ** 40), enc_seed=2, obj0=0)
        st.synchronize()
        ctxs.append(ctx); nets.append(C1Net(ctx, K, kb, W, b)); xs.append(x); streams.append(st)

    def run(n_ctx, steps):
        for w in range(4):
            nets[w % n_ctx].forward(xs[w % n_ctx])
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(streams[0])
        for k in range(1, n_ctx):
            streams[k].wait_event(e0)
        for s in range(steps):
            nets[s % n_ctx].forward(xs[s % n_ctx])
        for k in range(1, n_ctx):
            j = torch.cuda.Event()
            j.record(streams[k])
            streams[0].wait_event(j)
        e1.record(streams[0])
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / steps

    res = {}
    for rep in range(2):
        for nc in (1, 2, 3):
            res[f"ctx{nc}_ms_{rep}"] = run(nc, steps)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
