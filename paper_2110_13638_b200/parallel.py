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


def ct_slice(arr, start: int, stop: int, n: int):
    """Ciphertexts [start, stop) of a CtArray as a view (layout [count][2][level+1][N])."""
    from .edl import CtArray
    w = 2 * (arr.level + 1) * n
    return CtArray(arr.tensor[start * w:stop * w], stop - start, arr.level, arr.scale, arr.key_id)


def gather_cts(ctx, full, idx: Sequence[int]):
    """New array holding ciphertexts full[idx] (device gather; setup, not the hot path)."""
    import torch
    from .edl import CtArray
    w = 2 * (full.level + 1) * ctx.n
    t = full.tensor.view(full.count, w).index_select(0, torch.as_tensor(list(idx), device=full.tensor.device))
    return CtArray(t.reshape(-1).contiguous(), len(idx), full.level, full.scale, full.key_id)


def rank_inputs(ctx, sharded, full_batches):
    """This rank's strip array from full per-batch pixel arrays (784 cts each)."""
    import torch
    from .edl import CtArray
    parts = [gather_cts(ctx, full_batches[bi], sharded.pixels(bi)) for bi in range(sharded.batches)]
    f = full_batches[0]
    return CtArray(torch.cat([p.tensor for p in parts]), sum(p.count for p in parts), f.level, f.scale, f.key_id)


class ShardedCNN:
    """Per-rank C4 driver over the C-ABI (edl.Context).

    The rank's input is ONE ciphertext array holding, batch after batch, the strips of its
    windows (16 pixel ciphertexts per window, `strip_pixels` order).  One step:
      * cross-correlation per batch strip into one [batch][filter][window] array,
      * sigma_a once over all of the rank's 5 x 49 CC outputs (full-size launches),
      * dense partial sums (no rescale) per batch into partials[b] (zeros if the rank
        holds no window of batch b),
      * ONE uint64 all-reduce of partials [B][10][2][2][N] over NCCL (the exchange step),
      * per-limb mod q + rescale + bias of the batches this rank finishes (b = rank mod R).
    Bit-identical to the unsharded network (O4, O15)."""

    def __init__(self, ctx, K, kb, W, b, world: int, rank: int, batches: int):
        self.ctx, self.K, self.kb, self.W, self.b = ctx, K, kb, W, b
        self.world, self.rank, self.batches = world, rank, batches
        self.ranges = rank_windows(world, rank, batches)
        self.nw = [w1 - w0 for w0, w1 in self.ranges]
        self.woff = list(np.cumsum([0] + self.nw[:-1]))
        self.units = int(sum(self.nw))
        self.Wc = [np.ascontiguousarray(W[:, dense_columns(w0, w1)]) for w0, w1 in self.ranges]
        self.mine = [bi for bi in range(batches) if bi % world == rank]

    def pixels(self, batch: int) -> List[int]:
        return strip_pixels(*self.ranges[batch])

    def input_pixels(self) -> List[Tuple[int, int]]:
        """(batch, pixel) of every input ciphertext of this rank, in array order."""
        return [(bi, px) for bi in range(self.batches) for px in self.pixels(bi)]

    def partials_words(self, level: int = 1) -> int:
        return self.batches * 10 * 2 * (level + 1) * self.ctx.n

    def partials(self, x, out_tensor):
        """x: this rank's strips (16 * units ciphertexts, level 4).  Writes the un-rescaled
        dense partial of each batch into out_tensor[b]; returns (level, scale)."""
        c, n = self.ctx, self.ctx.n
        F = self.K.shape[0]
        cc = c.empty(F * self.units, max(x.level - 1, 0))
        for bi in range(self.batches):
            if self.nw[bi] == 0:
                continue
            xs = ct_slice(x, 16 * self.woff[bi], 16 * (self.woff[bi] + self.nw[bi]), n)
            dst = ct_slice(cc, F * self.woff[bi], F * (self.woff[bi] + self.nw[bi]), n)
            r = c.cross_correlate(xs, 4, 4 * self.nw[bi], self.K, 4, self.kb, out=dst)
            cc.level, cc.scale, cc.key_id = r.level, r.scale, r.key_id
        act = c.poly_activation(cc, (0.5, 0.197, 0.0, -0.004))
        words = out_tensor.numel() // self.batches
        meta = (act.level, act.scale * float(c.params.qs[act.level]))
        for bi in range(self.batches):
            dst = out_tensor[bi * words:(bi + 1) * words]
            if self.nw[bi] == 0:
                dst.zero_()
                continue
            a = ct_slice(act, F * self.woff[bi], F * (self.woff[bi] + self.nw[bi]), n)
            part = c.dense(a, self.Wc[bi], None, defer_rescale=True, out=c.wrap(dst, 10, act.level))
            meta = (part.level, part.scale)
        return meta

    def finish(self, summed_tensor, level: int, scale: float, batches=None):
        """After the uint64 all-reduce: mod q, rescale, bias of `batches` (default: this
        rank's) -> {batch: output array (10 ciphertexts)}."""
        c = self.ctx
        words = summed_tensor.numel() // self.batches
        outs = {}
        for bi in (self.mine if batches is None else batches):
            acc = c.wrap(summed_tensor[bi * words:(bi + 1) * words], 10, level, scale)
            c.mod_reduce(acc)
            outs[bi] = c.dense_finish(acc, self.b)
        return outs

    def step(self, x, partial_tensor, all_reduce: Callable):
        lvl, sc = self.partials(x, partial_tensor)
        if self.world > 1:
            all_reduce(partial_tensor)
        return self.finish(partial_tensor, lvl, sc)
