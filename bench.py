"""Benchmark: encrypted images/s of the C1 CNN (BASELINE.json configs[1]) on B200.

One step = server-side homomorphic inference of one 8192-image batch (784 pixel
ciphertexts at level 4 resident in HBM -> CC 5x4x4/4 -> sigma_a -> dense 245->10), i.e.
every row of SURVEY §8(a) a2-a10.  `value` is device-timed (CUDA events on the library's
stream, barrier + synchronize on both sides, max over ranks); `e2e` repeats the step
through the public API with the inputs copied from pinned host memory and the 10 output
ciphertexts copied back inside the timed region.  N>1: each rank runs its own batch
(weak scaling, independent batches -- the path needs no collective for them).

`--impl reference` times the oracle (oracle/, the plain CPU implementation) on the same
workload on the host cores -- every step one full 8192-image batch, its 49 CC windows
spread over one single-threaded process per core -- and prints the same JSON line (same
metric, unit and config).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "encrypted images/s (CKKS N=2^14 CNN)"
UNIT = "images/s"
BATCH = 8192
WINDOWS = 49


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=12)
    ap.add_argument("--cpu-windows", type=int, default=8, help="single-core oracle sample (windows of 49)")
    ap.add_argument("--cpu-procs", type=int, default=0, help="oracle processes (0: one per core, <= 49)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-c2", action="store_true", help="skip the C2 microbench sweep")
    ap.add_argument("--no-c3", action="store_true", help="skip the C3 tabular net")
    ap.add_argument("--inflight", type=int, default=4,
                    help="N=1: batches in flight (consecutive steps alternate over this many contexts, each "
                         "with its own stream pair and scratch); 1 = one batch at a time")
    return ap.parse_args()


def c1_config(world: int) -> dict:
    """The workload dict both arms print (same_config)."""
    return {"workload": ("C1 Fashion-MNIST-shaped encrypted CNN, CKKS N=2^14 {60,40,40,40,40|60}, "
                         "batch 8192 in slots (784 pixel ciphertexts), CC 5x4x4/4 -> sigma_a -> "
                         "dense 245->10") if world == 1 else
                        (f"C4 scale-out CNN: {world} batches of 8192 synthetic images (C1 "
                         f"architecture and parameters), 49*{world} (window, batch) units over "
                         f"{world} GPUs"), "global_batch": BATCH * world,
            "parallelism": ("single GPU" if world == 1 else
                            f"C4 (window, batch) units sharded x{world}, NCCL uint64 all-reduce of "
                            f"dense partials"),
            "l2": "inputs 1.03 GB per GPU > L2 (no flush)"}


def cpu_info() -> dict:
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cpu_model": model, "numpy": np.__version__, "host_cores": len(os.sched_getaffinity(0))}


# ----------------------------------------------------------------------------- oracle sample
def oracle_sample_seconds(windows: int, seed_data: int = 2110):
    """Oracle (CPU) server-side inference restricted to `windows` of the 49 CC windows:
    CC for those windows (5 filters each), sigma_a on those 5*windows ciphertexts, dense
    partial sums over them into the 10 outputs, final rescale + bias.  Work scales
    linearly in windows (the final 10-ciphertext rescale is <0.1%)."""
    from oracle import layers, networks
    from oracle.ckks import CtArray
    from synth import c1_images, c1_slots, c1_weights

    K, kb, W, b = c1_weights()
    imgs = c1_images(BATCH, seed_data)
    slots = c1_slots(imgs)
    ctx = networks.c1_context(1)
    wins = list(range(windows))
    pix = sorted({(4 * (w // 7) + u) * 28 + 4 * (w % 7) + v for w in wins for u in range(4) for v in range(4)})
    polys = np.stack([ctx.encode(slots[p]) for p in pix])
    xs = ctx.encrypt_poly(polys, 2, 0, ctx.p.scale)
    full = np.zeros((784, 2, 5, ctx.n), dtype=np.uint64)
    full[pix] = xs.data
    x = CtArray(full, 4, xs.scale, xs.key_id)
    t0 = time.perf_counter()
    # CC restricted to the sampled windows
    cc_parts = []
    for f in range(5):
        for w in wins:
            r, c = divmod(w, 7)
            idx = [(4 * r + u) * 28 + 4 * c + v for u in range(4) for v in range(4)]
            cc_parts.append(layers.weighted_sum(ctx, x, idx, [K[f, u, v] for u in range(4) for v in range(4)],
                                                float(ctx.q[4])))
    acc = CtArray(np.stack(cc_parts), 4, x.scale * float(ctx.q[4]), x.key_id)
    cc = ctx.add_scalar(ctx.rescale(acc), np.repeat(kb, len(wins)))
    act = layers.poly_activation(ctx, cc, networks.SIGMA_A)
    cols = [f * WINDOWS + w for f in range(5) for w in wins]
    out = layers.dense(ctx, act, W[:, cols], b)
    t = time.perf_counter() - t0
    assert out.count == 10
    return t


def _oracle_shard(conn, windows, seed_data):
    """One single-threaded host process: the oracle's C1 step restricted to `windows` (CC of
    those windows for the 5 filters, sigma_a on their 5*len(windows) outputs, the dense
    layer's un-rescaled partial sums over them).  Setup (keys, encryption) happens once;
    every "go" runs the step and returns (t_start, t_end, partial accumulators)."""
    from oracle import layers, networks
    from oracle.ckks import CtArray
    from synth import c1_images, c1_slots, c1_weights

    K, kb, W, b = c1_weights()
    ctx = networks.c1_context(1)
    slots = c1_slots(c1_images(BATCH, seed_data))
    pix = [(4 * (w // 7) + u) * 28 + 4 * (w % 7) + v for w in windows for u in range(4) for v in range(4)]
    xs = [ctx.encrypt_poly(ctx.encode(slots[p])[None, :], 2, p, ctx.p.scale) for p in pix]   # object id = pixel
    x = CtArray(np.concatenate([c.data for c in xs]), 4, xs[0].scale, xs[0].key_id)
    cols = [f * WINDOWS + w for f in range(5) for w in windows]
    ql = float(ctx.q[4])
    conn.send("ready")
    while conn.recv() == "go":
        t0 = time.time()
        parts = [layers.weighted_sum(ctx, x, range(16 * k, 16 * k + 16), K[f].reshape(-1), ql)
                 for f in range(5) for k in range(len(windows))]
        cc = ctx.add_scalar(ctx.rescale(CtArray(np.stack(parts), 4, x.scale * ql, x.key_id)),
                            np.repeat(kb, len(windows)))
        act = layers.poly_activation(ctx, cc, networks.SIGMA_A)
        part = layers.dense_partial(ctx, act, W[:, cols])
        conn.send((t0, time.time(), part.data, part.level, part.scale))


class OracleFullBatch:
    """The oracle on one full 8192-image C1 batch per step, its 49 windows split over P
    single-threaded processes (one per host core, P <= 49); the per-process dense partials
    are combined exactly as the multi-GPU path does (uint64 sum, mod q, rescale, bias:
    oracle.layers.combine_partials / dense_finish).  Step time = last finish - first start
    (host clock), setup excluded."""

    def __init__(self, procs: int):
        import multiprocessing as mp
        os.environ.setdefault("OMP_NUM_THREADS", "1")
        cores = len(os.sched_getaffinity(0))
        self.P = max(1, min(WINDOWS, procs if procs > 0 else cores))
        chunks = [list(range(WINDOWS))[k::self.P] for k in range(self.P)]
        mpc = mp.get_context("spawn")
        self.conns, self.procs = [], []
        for ch in chunks:
            a, b = mpc.Pipe()
            p = mpc.Process(target=_oracle_shard, args=(b, ch, 2110), daemon=True)
            p.start()
            self.conns.append(a)
            self.procs.append(p)
        for c in self.conns:
            assert c.recv() == "ready"

    def step(self):
        from oracle import layers, networks
        from oracle.ckks import CtArray
        from synth import c1_weights
        for c in self.conns:
            c.send("go")
        res = [c.recv() for c in self.conns]
        t = max(r[1] for r in res) - min(r[0] for r in res)
        if not hasattr(self, "_fin"):
            self._fin = networks.c1_context(1)
        ctx = self._fin
        parts = [CtArray(r[2], r[3], r[4], ctx.key_id) for r in res]
        out = layers.dense_finish(ctx, layers.combine_partials(ctx, parts), c1_weights()[3])
        assert out.count == 10 and out.level == 0
        return t

    def close(self):
        for c in self.conns:
            c.send("stop")
        for p in self.procs:
            p.join(timeout=10)


def run_reference(a):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    ob = OracleFullBatch(a.cpu_procs)
    nb = max(a.gpus, 1)   # N > 1: the C4 step is N batches (global_batch 8192 N), run one after the other
    for _ in range(max(a.warmup, 0)):
        ob.step()
    per_step = [sum(ob.step() for _ in range(nb)) for _ in range(a.steps)]
    ob.close()
    t_full = float(np.mean(per_step))
    value = nb * BATCH / t_full
    sample = (f"every step {nb} full 8192-image C1 batch(es) (all 49 CC windows, sigma_a on 245 ciphertexts, "
              f"dense 245->10 incl. rescale + bias), no extrapolation; {ob.P} single-threaded oracle processes")
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup,
            "ms_per_step": t_full * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "u64", "data": "synthetic", "impl": "reference",
            "config": c1_config(nb),
            "cpu_baseline": dict({"value": value, "unit": UNIT, "cores": ob.P, "kind": "oracle", "sample": sample},
                                 **cpu_info()),
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        rows = [r for r in self.rows if len(r) >= 7]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[3 + k].lower().startswith("active")})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# ----------------------------------------------------------------------------- algorithmic work
# Limb transforms of one C1 step per NTT-family kernel, split by arithmetic path: "int" =
# the 60-bit primes (q0, P: Shoup butterflies), "fp" = the 40-bit primes (q1..q4: FP64-
# quotient butterflies).  From the schedule: CC rescale at l=4 (245 cts),
# sigma_a on 245 cts (relin + rescale at l=3, scalar rescales of u and w, relin + rescale
# at l=2), dense rescale at l=1 (10 cts).  Each transform is (N/2) log2 N butterflies.
C1_TRANSFORMS = {
    #                        (int,  fp)
    "k_rescale_intt":       (0, 490 + 490 + 20),
    "k_rescale_ntt":        (490 + 490 + 490 + 20, 1470 + 980 + 490),
    "k_relin_intt_d2":      (245 + 245, 735 + 490),
    "k_relin_modup":        (245 * 7 + 245 * 5, 245 * 9 + 245 * 4),
    "k_relin_ks":           (245 * 7 + 245 * 5, 245 * 9 + 245 * 4),   # fused variant (EDL_KS_FUSED=1)
    "k_relin_moddown_intt": (490 + 490, 490 + 490),
    "k_relin_moddown_ntt":  (490 + 490, 980 + 490),
}


# Algorithmic HBM bytes of one C1 step per kernel (all its launches in the step): every
# operand limb read once, every output limb written once, 2^14 x 8 B per limb; keys and
# constants (L2-resident) not counted.  Derivation per kernel in DESIGN.md §5.
_LIMB = 8 << 14
C1_ALG_LIMBS = {
    "k_cc_mac": 784 * 2 * 5 + 245 * 2 * 5,                          # 784 cts in @l=4, 245 out @l=4
    "k_rescale_intt": (490 + 490) + (490 + 980) + (20 + 20),         # CC l=4; sigma u/w shared INTT (2 outs); dense
    "k_rescale_ntt": (1960 + 490 + 1960) + (1470 + 490 + 1470) + (980 + 490 + 980) + (20 + 20 + 20),
    "k_relin_intt_d2": (980 + 980) + (1470 + 735),                  # y*y (a == b) l=3; u*y2 l=2
    "k_relin_modup": (980 + 3920) + (735 + 2205),                   # digits in, (l+1)^2 raised limbs out
    "k_relin_mac": (3920 + 1960 + 2450) + (2205 + 2940 + 1960),     # raised digits + tensor operands in, acc out
    "k_relin_ks": (980 + 1960 + 2450) + (735 + 2940 + 1960),        # fused: digits + tensor operands in, acc out
    "k_relin_moddown_intt": 1960 + 1960,
    "k_relin_moddown_ntt": (490 + 490 + 1470 + 1470) + (490 + 490 + 980 + 980 + 980),
    "k_dense_mac": 980 + 40,
}
C1_ALG_BYTES = {k: v * _LIMB for k, v in C1_ALG_LIMBS.items()}

# Modular MACs of one C1 step per MAC kernel, (F64-path 40-bit limbs, 60-bit limbs): CC
# 245 outputs x 16 taps x 2 polys x N on q1..q4 | q0; dense 245 x 10 x 2 x N on q1 | q0; key
# products per (ciphertext, target, coefficient): 2 (l+1) key MACs + the tensor's 4 products
# on data targets (q0 and P are the 60-bit targets), l = 3 and l = 2.
_N14 = 1 << 14
C1_MACS = {
    "k_cc_mac": (245 * 16 * 2 * 4 * _N14, 245 * 16 * 2 * 1 * _N14),
    "k_dense_mac": (245 * 10 * 2 * _N14, 245 * 10 * 2 * _N14),
    "k_relin_mac": (245 * _N14 * (3 * 12 + 2 * 10), 245 * _N14 * ((12 + 8) + (10 + 6))),
}
# k_cc_mac4 (round 2b) runs its F64-limb MACs as exact 22-bit split products: 4 DFMA per MAC,
# + 2 DADD per tap for the split of x shared by 5 filters (0.4), + ~21 FP64 instructions per
# output to fold the three sums (S0 mod q + S1 2^22 + S2 2^44) over 16 taps (1.3): its F64
# ceiling is the measured DFMA rate / 5.7 instead of the f64_mulc-MAC probe.
C1_F64_DP_PER_MAC = {"k_cc_mac": 4.0 + 2.0 / 5 + 21.0 / 16}


def ntt_roofline(name, ms_total, steps, n, peak_int, peak_fp):
    """Achieved algorithmic butterflies/s of one NTT-family kernel over the timed region
    against the register-only butterfly ceiling for its mix of primes."""
    ti, tf = C1_TRANSFORMS[name]
    bfly = (n // 2) * (n.bit_length() - 1)
    work = (ti + tf) * bfly * steps
    peak_mix = (ti + tf) / (ti / peak_int + tf / peak_fp)
    achieved = work / (ms_total / 1e3)
    return achieved, peak_mix


# ----------------------------------------------------------------------------- ours
def run_ours(a):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # EDL_BENCH_EMULATE=1 (functional check of the N>1 path on a one-GPU box, never a
    # timing): every rank on cuda:0, gloo all-reduce through the host
    emulate = os.environ.get("EDL_BENCH_EMULATE") == "1"
    if emulate:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if emulate:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_2110_13638_b200 import edl, parallel
    from paper_2110_13638_b200.networks import C1Net
    from synth import c1_images, c1_slots, c1_weights

    stream = torch.cuda.Stream(device=local)
    torch.cuda.set_stream(stream)
    ctx = edl.Context(edl.params_from_depth(4), device=local, stream=stream).keygen(1)
    K, kb, W, b = c1_weights()
    if world == 1:
        # C1: one 8192-image batch, the paper's graph engine firing CC -> sigma_a -> dense
        imgs = c1_images(BATCH, 2110)
        polys = torch.from_numpy(ctx.encode(c1_slots(imgs))).to(f"cuda:{local}")
        x = ctx.encrypt_poly(polys, scale=float(2 ** 40), enc_seed=2, obj0=0)
        # the same images as secret-key ciphertexts for the seeded wire format (e2e)
        x_sk = ctx.encrypt_poly_sk(polys, scale=float(2 ** 40), enc_seed=3, obj0=0)
        del polys
        net = C1Net(ctx, K, kb, W, b)

        def step(inp):
            return net.forward(inp)["out"]

        # Batches in flight (serving pipeline): consecutive steps alternate over `inflight`
        # contexts -- same keys (same seed), own stream pair and scratch, own resident batch of
        # images -- so the head of batch k+1 (CC, rescale) fills the SMs that the tail of batch k
        # (last key-switch waves, dense MAC, 10-ciphertext rescale) leaves idle.  Every step is
        # still one full 8192-image batch through the whole path.
        pipe = [(ctx, net, x, stream)]
        for i in range(1, max(1, a.inflight)):
            st_i = torch.cuda.Stream(device=local)
            with torch.cuda.stream(st_i):
                ctx_i = edl.Context(edl.params_from_depth(4), device=local, stream=st_i).keygen(1)
                polys_i = torch.from_numpy(ctx_i.encode(c1_slots(c1_images(BATCH, 2110 + i)))).to(f"cuda:{local}")
                x_i = ctx_i.encrypt_poly(polys_i, scale=float(2 ** 40), enc_seed=2, obj0=784 * i)
                del polys_i
            st_i.synchronize()
            pipe.append((ctx_i, C1Net(ctx_i, K, kb, W, b), x_i, st_i))

        def step_pipe(k):
            c_k, net_k, x_k, st_k = pipe[k % len(pipe)]
            with torch.cuda.stream(st_k):   # torch allocations of this step on the step's stream
                return net_k.forward(x_k)["out"]
    else:
        # C4 (configs[4]) at weak scale: `world` batches of 8192 images, their 49*world
        # (window, batch) units split over the ranks (49 each), dense partials combined by
        # one NCCL uint64 all-reduce, each rank finishing one batch
        sh = parallel.ShardedCNN(ctx, K, kb, W, b, world, rank, world)
        # each rank encrypts only its own strip ciphertexts (16 per (window, batch) unit; object
        # id = batch * 784 + pixel, as an unsharded encryption of that batch would use)
        strips = []
        for bi in range(world):
            px = sh.pixels(bi)
            if not px:
                continue
            sl = c1_slots(c1_images(BATCH, 2110 + bi))[px]
            polys = torch.from_numpy(ctx.encode(sl)).to(f"cuda:{local}")
            for k, p in enumerate(px):
                strips.append(ctx.encrypt_poly(polys[k:k + 1], scale=float(2 ** 40), enc_seed=2, obj0=784 * bi + p))
            del polys
        x = edl.CtArray(torch.cat([s_.tensor for s_ in strips]), len(strips), 4, strips[0].scale, strips[0].key_id)
        x_sk = None   # rank inputs are strips: the e2e at N > 1 uses the public-key wire
        del strips
        torch.cuda.empty_cache()
        nccl_v = getattr(torch.cuda.nccl, "version", lambda: None)()
        print(f"bench rank {rank}/{world}: backend {dist.get_backend()} NCCL {nccl_v} device cuda:{local} "
              f"({torch.cuda.get_device_name(local)}), {sh.units} (window, batch) units, "
              f"{x.count} input ciphertexts ({x.tensor.numel() * 8 / 2**30:.2f} GiB)", file=sys.stderr, flush=True)
        partials = torch.empty(sh.partials_words(), dtype=torch.int64, device=f"cuda:{local}")

        def all_reduce(t):
            dist.all_reduce(t, op=dist.ReduceOp.SUM)   # int64 two's-complement sum == uint64 sum

        def step(inp):
            outs = sh.step(inp, partials, all_reduce)
            return outs[rank]

    def barrier():
        if world > 1:
            dist.barrier()

    piped = world == 1 and len(pipe) > 1
    for _ in range(max(a.warmup, 0)):
        step(x)
        if piped:
            for j in range(1, len(pipe)):
                step_pipe(j)
    torch.cuda.synchronize(local)
    barrier()

    clocks = ClockSampler(local)
    clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ms_one = None
    if piped:
        # one batch at a time first (the latency of a batch, reported beside the pipelined rate)
        e0.record(stream)
        for _ in range(a.steps):
            out = step(x)
        e1.record(stream)
        stream.synchronize()
        ms_one = e0.elapsed_time(e1) / a.steps
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = sum(p_[0].launches for p_ in pipe) if world == 1 else ctx.launches
    torch.cuda.synchronize(local)
    barrier()
    e0.record(stream)
    if piped:
        for p_ in pipe[1:]:
            p_[3].wait_event(e0)
        for k in range(a.steps):
            out = step_pipe(k)
        for p_ in pipe[1:]:
            j_ = torch.cuda.Event()
            j_.record(p_[3])
            stream.wait_event(j_)
    else:
        for _ in range(a.steps):
            out = step(x)
    e1.record(stream)
    torch.cuda.synchronize(local)
    barrier()
    ms = e0.elapsed_time(e1)
    launches = (sum(p_[0].launches for p_ in pipe) if world == 1 else ctx.launches) - l0
    clk = clocks.stop()
    # per-kernel durations (roofline, kernel split): the same K steps again with a CUDA event
    # pair around every launch on the library's stream; the events' own gaps would inflate the
    # step, so `value` comes from the clean pass above
    ctx.profile(True)
    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    stream.synchronize()
    barrier()
    p0.record(stream)
    for _ in range(a.steps):
        step(x)
    p1.record(stream)
    stream.synchronize()
    barrier()
    ms_instr = p0.elapsed_time(p1)
    prof = ctx.profile_read()
    ctx.profile(False)
    t = torch.tensor([ms], dtype=torch.float64, device=f"cuda:{local}")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    ms_step = ms_max / a.steps
    value = world * BATCH * a.steps / (ms_max / 1e3)

    # ---- e2e: same step through the public API with host buffers.  Every step copies its
    # input ciphertexts from pinned host memory and reads its 10 output ciphertexts back;
    # the host->device copy of step k+1 runs on a copy stream while step k computes (two
    # device input buffers), so the pipeline is bound by the slower of PCIe and compute.
    e2e = None
    if not a.no_e2e:
        out_words = out.tensor.numel()
        host_out = [torch.empty(out_words, dtype=torch.int64, pin_memory=True) for _ in range(2)]
        dev_in = [edl.CtArray(torch.empty_like(x.tensor), x.count, x.level, x.scale, x.key_id) for _ in range(2)]

        def measure_e2e(host_in, unpack_host):
            """Every step through the C-ABI's host-buffer calls: edl_wire_upload (pinned host bytes ->
            the context's staging slot, on the context's copy stream), edl_cts_unpack*_host (the
            compute stream waits for the slot, unpacks), the step, edl_cts_download (outputs ->
            pinned host memory).  The upload of step k+1 is queued while step k computes."""
            def run_pipeline(nsteps, first_event=None):
                for k in range(nsteps):
                    buf = k % 2
                    if k == 0 and first_event is not None:
                        first_event.record(stream)
                    ctx.wire_upload(buf, host_in)
                    unpack_host(buf, dev_in[buf])
                    res = step(dev_in[buf])
                    ctx.download(res, host_out[buf])

            run_pipeline(2)
            ctx.sync()
            barrier()
            f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            run_pipeline(a.e2e_steps, first_event=f0)
            f1.record(stream)
            ctx.sync()
            barrier()
            te = torch.tensor([f0.elapsed_time(f1)], dtype=torch.float64, device=f"cuda:{local}")
            if world > 1:
                dist.all_reduce(te, op=dist.ReduceOp.MAX)
            return world * BATCH * a.e2e_steps / (float(te.item()) / 1e3)

        def pinned(t):
            h = torch.empty(t.numel(), dtype=torch.int64, pin_memory=True)
            h.copy_(t.cpu())
            return h

        # public-key ciphertexts in the packed wire format (edl.h: residues in bit-length-of-q bits)
        host_pk = pinned(ctx.pack(x))
        v_pk = measure_e2e(host_pk, lambda sl, o: ctx.unpack_host(sl, x.count, x.level, x.scale, x.key_id, out=o))
        e2e_pk = {"value": v_pk, "unit": UNIT, "h2d_bytes_per_step": int(host_pk.numel() * 8),
                  "d2h_bytes_per_step": int(out_words * 8),
                  "inputs": "public-key ciphertexts, packed wire format (edl_cts_pack/unpack)"}
        del host_pk
        pipeline = ("C-ABI host-buffer calls: edl_wire_upload of step k+1 (pinned host memory -> the context's "
                    "staging slot on its copy stream) overlaps step k; edl_cts_unpack*_host, the step's kernels and "
                    "edl_cts_download of the 10 output ciphertexts to pinned host memory inside the timed region")
        if x_sk is not None:
            # secret-key ciphertexts of the same images (reading Z16): c0 packed, c1 regenerated on the
            # device from (enc_seed, object id) by edl_cts_unpack_seeded inside each step
            host_sk = pinned(ctx.pack_c0(x_sk))
            v_sk = measure_e2e(host_sk, lambda sl, o: ctx.unpack_seeded_host(sl, x_sk.count, x_sk.level, x_sk.scale,
                                                                              x_sk.key_id, enc_seed=3, obj0=0, out=o))
            e2e = {"value": v_sk, "unit": UNIT, "h2d_bytes_per_step": int(host_sk.numel() * 8),
                   "d2h_bytes_per_step": int(out_words * 8),
                   "inputs": "secret-key ciphertexts of the same 8192 images (DESIGN reading Z16): c0 in the "
                             "packed wire format, c1 regenerated on the device from the 8-byte seed",
                   "pipeline": pipeline, "public_key": e2e_pk,
                   "unpacked_bytes_per_step": int(x.tensor.numel() * 8)}
            del host_sk
        else:
            e2e = dict(e2e_pk, pipeline=pipeline, unpacked_bytes_per_step=int(x.tensor.numel() * 8))

    # ---- roofline: every kernel against BOTH ceilings -- measured HBM (MEASURED_PEAKS.json)
    # and, for the NTT family, the measured butterfly ceiling of its prime mix -- and the
    # dominant kernel (largest share of the instrumented step) in the contract's keys
    n = ctx.n
    dom = max(prof.items(), key=lambda kv: kv[1][0]) if prof else ("none", (0.0, 0))
    peak_int = ctx.bfly_peak(0)          # q0 (60-bit): Shoup path
    peak_fp = ctx.bfly_peak(1)           # q1 (40-bit): FP64-pipe path
    dfma = ctx.pipe_peak(0)              # raw FP64 pipe: DFMA lane-ops/s
    imadw = ctx.pipe_peak(1)             # raw integer multiply: IMAD.WIDE.U32 lane-ops/s
    fmac = ctx.pipe_peak(2)              # F64 modular MAC (40-bit limbs of the MAC layers) / s
    imac = ctx.pipe_peak(3)              # 128-bit lazy MAC (60-bit limbs) / s
    sms = torch.cuda.get_device_properties(local).multi_processor_count
    nominal_dp = sms * 64 * 1965e6       # 64 FP64 lanes / SM / clk at the max SM clock
    hbm_peak = None
    try:
        hbm_peak = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
        hbm_kind = "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        hbm_peak, hbm_kind = 6650.0, "fallback (B200_PROFILING.md)"
    traffic_tab = {}
    tf = os.path.join(ROOT, "profiles", "round2", "ncu_traffic.json")
    if os.path.exists(tf):
        traffic_tab = json.load(open(tf))
    per_kernel = {}
    if world == 1:
        for name, (ms_tot, cnt) in prof.items():
            ms_k = ms_tot / a.steps
            e = {"ms_per_step": ms_k, "launches_per_step": cnt / a.steps, "share_of_step": ms_tot / ms_instr}
            if name in C1_ALG_BYTES:
                gbs = C1_ALG_BYTES[name] / (ms_k / 1e3) / 1e9
                e.update({"alg_bytes_per_step": C1_ALG_BYTES[name], "hbm_GBps": gbs, "hbm_frac": gbs / hbm_peak})
            if name in C1_TRANSFORMS:
                ach, pk = ntt_roofline(name, ms_tot, a.steps, n, peak_int, peak_fp)
                e.update({"achieved_Gbfly_s": ach / 1e9, "peak_Gbfly_s": pk / 1e9, "bfly_frac": ach / pk})
            if name in C1_MACS:   # MAC layers: time at the measured MAC ceilings / measured time
                nf, ni = C1_MACS[name]
                fceil = dfma / C1_F64_DP_PER_MAC[name] if name in C1_F64_DP_PER_MAC else fmac
                t_peak = nf / fceil + ni / imac
                e.update({"macs_per_step": nf + ni, "mac_alu_frac": t_peak / (ms_k / 1e3)})
            fr = {"hbm": e.get("hbm_frac", 0.0), "alu": e.get("bfly_frac", e.get("mac_alu_frac", 0.0))}
            e["bound"] = max(fr, key=fr.get) if any(fr.values()) else None
            tk = name if name in traffic_tab else next((k for k in traffic_tab if k.startswith(name)), None)
            if tk is not None:   # ncu names the template (k_cc_mac4), the library the launch (k_cc_mac)
                e["dram_bytes_per_step_ncu"] = traffic_tab[tk]["dram_bytes_per_step"]
            per_kernel[name] = e
    ntt_doms = [k for k in sorted(prof, key=lambda k: -prof[k][0]) if k in C1_TRANSFORMS]
    roof = None
    if ntt_doms and world == 1:
        k = ntt_doms[0]
        e = per_kernel[k]
        launches_k = e["launches_per_step"]
        traffic = None
        if k in traffic_tab:   # DRAM bytes of the kernel's launches in one step (ncu --set full) / launches
            traffic = traffic_tab[k]["dram_bytes_per_step"] / launches_k   # same divisor as the algorithmic bytes
        roof = {"kernel": k, "bound": "alu", "unit": "Gbutterfly/s", "achieved": e["achieved_Gbfly_s"],
                "peak": e["peak_Gbfly_s"], "frac": e["bfly_frac"], "traffic": traffic,
                "traffic_unit": "DRAM bytes per launch (profiles/round2/ncu_traffic.json: ncu --set full of "
                                "tools/prof_step.py, the bench step; bytes per step / launches per step)",
                "algorithmic_bytes_per_launch": C1_ALG_BYTES.get(k, 0) / launches_k,
                "hbm_frac": e.get("hbm_frac"), "hbm_peak_GBps": hbm_peak, "hbm_peak_kind": hbm_kind,
                "peak_kind": "measured: register-only Harvey CT butterflies (edl_bfly_peak) through the "
                             "kernel's own arithmetic paths, weighted by its 60-bit/40-bit transform mix",
                "peak_int_Gbfly_s": peak_int / 1e9, "peak_fp_Gbfly_s": peak_fp / 1e9,
                "pipe_anchor": {"dfma_lane_ops_per_s": dfma, "imad_wide_lane_ops_per_s": imadw,
                                "f64_mac_per_s": fmac, "mac128_per_s": imac,
                                "nominal_fp64_lane_ops_per_s": nominal_dp,
                                "fp_bfly_vs_dfma": peak_fp * 8 / dfma,
                                "note": "F64 butterfly = 8 FP64 instructions: peak_fp * 8 / dfma = the "
                                        "butterfly kernel's FP64-pipe efficiency"},
                "share_of_step": e["share_of_step"], "avg_launch_ms": prof[k][0] / prof[k][1],
                "largest_kernel_overall": dom[0]}
    kernels = {k: {"ms_per_step": v[0] / a.steps, "launches_per_step": v[1] / a.steps} for k, v in prof.items()}

    # ---- second half of BASELINE's metric: NTT limb-transforms/s (C2 shape at N = 2^14:
    # 256 ciphertexts x 2 polys x 5 limbs of the C1 chain, forward, device-timed)
    ntt_rate = None
    if rank == 0:
        nb = 256 * 2
        tl = torch.randint(0, 2 ** 39, (nb * 5 * n,), dtype=torch.int64, device=f"cuda:{local}")
        ctx.ntt_(tl, nb, 4, False)
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        stream.synchronize()
        g0.record(stream)
        for _ in range(5):
            ctx.ntt_(tl, nb, 4, False)
        g1.record(stream)
        stream.synchronize()
        ntt_rate = nb * 5 * 5 / (g0.elapsed_time(g1) / 1e3)
        del tl

    # ---- C4's companion series: replica data parallelism, one independent
    # 8192-image C1 batch per GPU and no communication, timed the same way (max over ranks)
    replica = None
    if world > 1:
        polys = torch.from_numpy(ctx.encode(c1_slots(c1_images(BATCH, 2110 + rank)))).to(f"cuda:{local}")
        xr = ctx.encrypt_poly(polys, scale=float(2 ** 40), enc_seed=2, obj0=0)
        del polys
        net_r = C1Net(ctx, K, kb, W, b)
        for _ in range(max(a.warmup, 1)):
            net_r.forward(xr)
        stream.synchronize()
        barrier()
        r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        r0.record(stream)
        for _ in range(a.steps):
            net_r.forward(xr)
        r1.record(stream)
        stream.synchronize()
        barrier()
        tr = torch.tensor([r0.elapsed_time(r1)], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(tr, op=dist.ReduceOp.MAX)
        replica = {"value": world * BATCH * a.steps / (float(tr.item()) / 1e3), "unit": UNIT,
                   "ms_per_step": float(tr.item()) / a.steps,
                   "config": f"{world} independent C1 batches (one per GPU), no communication"}
        del xr, net_r

    # ---- the other BASELINE configs, rank 0 at N = 1 (outside the timed C1 region):
    # C3 tabular net (configs[3]) and the C2 RNS microbench (configs[2]) at 3 and 24 limbs
    c3 = c2 = None
    if rank == 0 and world == 1:
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        if not a.no_c3:
            from c3_bench import run_c3
            c3 = run_c3(5, max(1, a.inflight))
            c3["config_index"] = 3
        if not a.no_c2:
            from c2_bench import point
            c2 = {"config_index": 2, "batch": 256, "unit": "NTT/INTT: M limb-transforms/s; key-switch/s",
                  "chains": "[60] + [40]*(L-2) + [60] data primes + one 60-bit special prime", "points": []}
            for logn in (13, 14, 15, 16):
                for L in (3, 24):
                    r = point(logn, L, 256, 3)
                    c2["points"].append({k: (round(v, 4) if isinstance(v, float) else v) for k, v in r.items()})
                    torch.cuda.empty_cache()

    props = torch.cuda.get_device_properties(local)
    device = {"name": props.name, "sms": props.multi_processor_count,
              "smem_per_sm_bytes": getattr(props, "shared_memory_per_multiprocessor", None),
              "l2_bytes": getattr(props, "L2_cache_size", None), "hbm_bytes": props.total_memory}

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        # all host cores: one full batch (no extrapolation), P single-threaded oracle processes
        ob = OracleFullBatch(a.cpu_procs)
        ob.step()                                   # warm-up
        t_all = min(ob.step() for _ in range(2))
        ob.close()
        # one core: a sample of the same step, extrapolated linearly in the number of windows
        ts = oracle_sample_seconds(a.cpu_windows)
        t1 = ts * WINDOWS / a.cpu_windows
        cpu = dict({"value": BATCH / t_all, "unit": UNIT, "cores": ob.P, "kind": "oracle",
                    "sample": f"one full 8192-image batch (49 CC windows over {ob.P} single-threaded oracle "
                              f"processes, dense partials combined), best of 2 after 1 warm-up, "
                              f"{t_all:.2f} s; no extrapolation",
                    "single_core": {"value": BATCH / t1, "unit": UNIT, "cores": 1,
                                    "sampled_s": ts, "sample": f"{a.cpu_windows} of 49 CC windows (CC + sigma_a + "
                                    f"dense partial over them) on one core",
                                    "extrapolation": f"x{WINDOWS / a.cpu_windows:.4g} (linear in windows)",
                                    "extrapolated_s_per_batch": t1}}, **cpu_info())

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
                "warmup": a.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "u64", "data": "synthetic",
                "config": c1_config(world),
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
                "clocks": clk, "dominant_kernel": dom[0], "kernels": per_kernel or kernels, "device": device,
                "kernel_timing": {"method": "CUDA event pair around every launch, on the library stream, over a "
                                            "second pass of the same K steps", "ms_per_step_instrumented":
                                  ms_instr / a.steps},
                "pipeline": ({"batches_in_flight": len(pipe), "ms_per_batch_one_at_a_time": ms_one,
                              "note": "consecutive steps alternate over contexts with their own stream pair, "
                                      "scratch and resident input batch; every step is one full batch; "
                                      "--inflight 1 times one batch at a time"} if world == 1 else None),
                "replica_dp": replica, "c2": c2, "c3": c3,
                "ntt_limb_transforms_per_s": {"value": ntt_rate, "config": "N=2^14, C1 chain limbs q0..q4, 256 "
                                              "ciphertexts x 2 polys, forward NTT, device-timed (outside the "
                                              "timed C1 region)"}}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    a = _args()
    if a.impl == "reference":
        return run_reference(a)
    return run_ours(a)


if __name__ == "__main__":
    sys.exit(main())
