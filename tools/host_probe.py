"""Is the C1 step host-bound?  Host enqueue time of one forward (no sync) against the device
time of the same step, and the device time of N back-to-back steps (the host runs ahead).
Also times the step captured once in a CUDA graph.  `EDL_LIB` selects a build."""
import json
import os
import sys
import time

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
    for _ in range(3):
        net.forward(x)
    torch.cuda.synchronize()
    res = {}
    enq = []
    for _ in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        net.forward(x)
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        enq.append(((t1 - t0) * 1e3, (t2 - t0) * 1e3))
    res["enqueue_ms_vs_wall_ms"] = [(round(a, 3), round(b_, 3)) for a, b_ in enq]
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(st)
    for _ in range(10):
        net.forward(x)
    e1.record(st)
    torch.cuda.synchronize()
    res["device_ms_per_step_10"] = round(e0.elapsed_time(e1) / 10, 4)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
