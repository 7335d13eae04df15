"""Eager vs CUDA-graph replay of one C1 step (the library's launches captured from its
stream, both of its streams joined inside): device-timed ms per step."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2110_13638_b200 import edl
from paper_2110_13638_b200.networks import C1Net
from synth import c1_images, c1_slots, c1_weights


def main():
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = edl.Context(edl.params_from_depth(4), stream=stream).keygen(1)
    K, kb, W, b = c1_weights()
    polys = torch.from_numpy(ctx.encode(c1_slots(c1_images(8192, 2110)))).cuda()
    x = ctx.encrypt_poly(polys, scale=float(2 ** 40), enc_seed=2, obj0=0)
    net = C1Net(ctx, K, kb, W, b)
    for _ in range(3):
        ref = net.forward(x)["out"]
    stream.synchronize()

    def timeit(fn, reps=10):
        a, bb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(reps):
            fn()
        bb.record(stream)
        stream.synchronize()
        return a.elapsed_time(bb) / reps

    eager = timeit(lambda: net.forward(x))
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        out = net.forward(x)["out"]
    g.replay()
    stream.synchronize()
    same = bool(torch.equal(out.tensor, ref.tensor))
    graph = timeit(g.replay)
    print(json.dumps({"eager_ms": eager, "graph_ms": graph, "graph_output_equal": same}))


if __name__ == "__main__":
    main()
