"""Hot-path networks of BASELINE.json's configs, fired through the paper's graph engine.

C0: dense 16->4 then x^2 (N=8192).  C1: CC 5x4x4/4 -> sigma_a -> dense 245->10
(N=16384, Fashion-MNIST shape).  C3: dense 32->64 -> sigma_a ->
dense 64->1 (tabular stand-in).  Each layer node's forward receptor
calls one C-ABI layer function; the chain graph is fired with Alg. 1-5 (graph.py).
"""
from __future__ import annotations

from typing import Dict

import numpy as np

from . import edl, graph

SIGMA_A = (0.5, 0.197, 0.0, -0.004)   # PAPER.md:407 (reading Z9: "+ -0.004x^3")
SQUARE = (0.0, 0.0, 1.0)


class _Sink:
    def __init__(self):
        self.value = None

    def __call__(self, s):
        self.value = s
        return None          # sinks emit nothing (Alg. 4 returns None -> no recursion)


def _run_chain(layers, x, keep: bool) -> Dict[str, edl.CtArray]:
    """layers: [(name, fn, cost)].  Fires x through input -> layers -> y_hat."""
    seen: Dict[str, edl.CtArray] = {}
    sink = _Sink()

    def wrap(name, fn):
        def f(s):
            out = fn(s)
            if keep:
                seen[name] = out
            return out
        return f

    nodes = [("x", lambda s: s, 0)] + [(n, wrap(n, f), c) for n, f, c in layers] + [("y_hat", sink, 0)]
    g = graph.chain(nodes)
    graph.fire(g, ["x"], ["forward"], [x])
    seen["out"] = sink.value
    return seen


class C0Net:
    """Tiny encrypted dense net: dense 16->4 (+bias) then x^2."""
    depth = 2

    def __init__(self, ctx: edl.Context, W: np.ndarray, b: np.ndarray):
        self.ctx, self.W, self.b = ctx, W, b

    def forward(self, x: edl.CtArray, keep: bool = False):
        c = self.ctx
        return _run_chain([("dense", lambda s: c.dense(s, self.W, self.b), 1),
                           ("act", lambda s: c.poly_activation(s, SQUARE), 1)], x, keep)


class C1Net:
    """Fashion-MNIST-shaped CNN in the batch-in-slots layout (one ciphertext per pixel)."""
    depth = 4

    def __init__(self, ctx: edl.Context, K, kb, W, b):
        self.ctx, self.K, self.kb, self.W, self.b = ctx, K, kb, W, b

    def forward(self, x: edl.CtArray, keep: bool = False):
        c = self.ctx
        return _run_chain([("cc", lambda s: c.cross_correlate(s, 28, 28, self.K, 4, self.kb), 1),
                           ("act", lambda s: c.poly_activation(s, SIGMA_A), 2),
                           ("dense", lambda s: c.dense(s, self.W, self.b), 1)], x, keep)


class C3Net:
    """Tabular regression net: dense 32->64, sigma_a, dense 64->1 (per slot-batch)."""
    depth = 4

    def __init__(self, ctx: edl.Context, W1, b1, W2, b2):
        self.ctx, self.W1, self.b1, self.W2, self.b2 = ctx, W1, b1, W2, b2

    def forward(self, x: edl.CtArray, keep: bool = False):
        c = self.ctx
        return _run_chain([("dense1", lambda s: c.dense(s, self.W1, self.b1), 1),
                           ("act", lambda s: c.poly_activation(s, SIGMA_A), 2),
                           ("dense2", lambda s: c.dense(s, self.W2, self.b2), 1)], x, keep)

    def forward_many(self, xs):
        """Several slot-batches in one pass: dense1 per batch into one array, sigma_a ONCE over
        all batches' hidden ciphertexts (the activation is per ciphertext, so the key switches
        run as one full-size launch sequence instead of one small one per batch), dense2 per
        batch.  Every output residue equals forward()'s (tests/test_gpu_full_configs.py)."""
        from .parallel import ct_slice
        c, n = self.ctx, self.ctx.n
        O1 = self.W1.shape[0]
        h = c.empty(O1 * len(xs), max(xs[0].level - 1, 0))
        for b, x in enumerate(xs):
            r = c.dense(x, self.W1, self.b1, out=ct_slice(h, O1 * b, O1 * (b + 1), n))
            h.level, h.scale, h.key_id = r.level, r.scale, r.key_id
        a = c.poly_activation(h, SIGMA_A)
        return [c.dense(ct_slice(a, O1 * b, O1 * (b + 1), n), self.W2, self.b2) for b in range(len(xs))]
