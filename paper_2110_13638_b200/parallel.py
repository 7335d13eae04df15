"""Multi-GPU sharding of the CNN (BASELINE.json configs[4], SURVEY §8(e) scheme 2).

Work units are (window, batch) pairs: 49 CC windows x B batches of 8192 images.  Units
are ordered window-major (u = w*B + b) and split contiguously over the ranks: every
rank gets 49*B/R units (balanced to one unit, unlike whole-window splits that cap 8-GPU
efficiency at 49/56), a unit's 16 pixel ciphertexts and 5 filter outputs never cross
ranks, and every batch's windows are spread over all ranks.  Each rank runs CC ->
sigma_a -> dense *partial* sums (no rescale) for its windows of every batch; the per-batch partials [B][10][2][2][N] are then combined by ONE uint64 sum over
NCCL (north_star: "dense layer's partial sums combined by one NCCL uint64 sum over
NVLink followed by a per-limb mod-q reduction (safe because 8 q < 2^64)") and finished
by mod-q reduction, rescale and bias (O15).  Bit-identical to the unsharded network.

The per-rank window strip is laid out as a 4 x (4 nw) image, so the unchanged
cross-correlation kernel (stride 4) produces the window outputs in [f][window] order.
"""
from __future__ import annotations

from typing import Callable, List, Sequence, Tuple

import numpy as np

WINDOWS = 49
GRID = 7          # 7 x 7 windows of 4 x 4 pixels on a 28 x 28 image


def rank_windows(world: int, rank: int, batches: int, windows: int = WINDOWS) -> List[Tuple[int, int]]:
    """Units u = w*batches + b split contiguously: rank gets [lo, hi).  For batch b its
    windows are {w : lo <= w*batches + b < hi} = [ceil((lo-b)/B), ceil((hi-b)/B))."""
    units = windows * batches
    lo = (units * rank) // world
    hi = (units * (rank + 1)) // world
    out = []
    for b in range(batches):
        w0 = max(0, -(-(lo - b) // batches))
        w1 = min(windows, -(-(hi - b) // batches))
        out.append((w0, max(w0, w1)))
    return out


def strip_pixels(w0: int, w1: int) -> List[int]:
    """Pixel indices (28x28 row-major) of windows [w0, w1) laid out as a 4 x 4(w1-w0) image."""
    out = []
    nw = w1 - w0
    for u in range(4):
        for k in range(nw):
            r, c = divmod(w0 + k, GRID)
            for v in range(4):
                out.append((4 * r + u) * 28 + 4 * c + v)
    return out


def dense_columns(w0: int, w1: int, filters: int = 5) -> List[int]:
    """Columns of W (245 = 5 filters x 49 windows, f-major) matching the strip's CC outputs."""
    return [f * WINDOWS + w for f in range(filters) for w in range(w0, w1)]


def combine(partials, all_reduce: Callable, mod_reduce: Callable):
    """Sum rank partials as uint64 (int64 two's complement wraps identically), then mod q."""
    all_reduce(partials)
    return mod_reduce(partials)


class ShardedCNN:
    """Per-rank C4 driver over the C-ABI (edl.Context)."""

    def __init__(self, ctx, K, kb, W, b, world: int, rank: int, batches: int):
        self.ctx, self.K, self.kb, self.W, self.b = ctx, K, kb, W, b
        self.world, self.rank, self.batches = world, rank, batches
        self.ranges = rank_windows(world, rank, batches)

    def pixels(self, batch: int) -> List[int]:
        return strip_pixels(*self.ranges[batch])

    def partials(self, xs: Sequence, out_tensor):
        """xs[b]: this rank's strip ciphertexts of batch b (16*nw_b cts, level 4) or None.
        Writes the un-rescaled dense partial of each batch into out_tensor[b] (zeros when
        the rank holds no window of that batch)."""
        c = self.ctx
        words = out_tensor.numel() // self.batches
        meta = None
        for bi, x in enumerate(xs):
            dst = out_tensor[bi * words:(bi + 1) * words]
            w0, w1 = self.ranges[bi]
            if w1 == w0:
                dst.zero_()
                continue
            Wc = np.ascontiguousarray(self.W[:, dense_columns(w0, w1)])
            cc = c.cross_correlate(x, 4, 4 * (w1 - w0), self.K, 4, self.kb)
            act = c.poly_activation(cc, (0.5, 0.197, 0.0, -0.004))
            part = c.dense(act, Wc, None, defer_rescale=True, out=c.wrap(dst, 10, act.level))
            meta = (part.level, part.scale)
        return meta

    def finish(self, summed_tensor, level: int, scale: float):
        """After the uint64 all-reduce: mod q, rescale, bias -> one output array per batch."""
        c = self.ctx
        words = summed_tensor.numel() // self.batches
        outs = []
        for bi in range(self.batches):
            acc = c.wrap(summed_tensor[bi * words:(bi + 1) * words], 10, level, scale)
            c.mod_reduce(acc)
            outs.append(c.dense_finish(acc, self.b))
        return outs
