"""Benchmark: encrypted images/s of the C1 CNN (BASELINE.json configs[1]) on B200.

One step = server-side homomorphic inference of one 8192-image batch (784 pixel
ciphertexts at level 4 resident in HBM -> CC 5x4x4/4 -> sigma_a -> dense 245->10), i.e.
every row of SURVEY §8(a) a2-a10.  `value` is device-timed (CUDA events on the library's
stream, barrier + synchronize on both sides, max over ranks); `e2e` repeats the step
through the public API with the inputs copied from pinned host memory and the 10 output
ciphertexts copied back inside the timed region.  N>1: each rank runs its own batch
(weak scaling, independent batches -- the path needs no collective for them).

`--impl reference` times the oracle (oracle/, the plain CPU implementation) on a bounded
sample of the same workload on the host cores and prints the same JSON line.
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
    ap.add_argument("--cpu-windows", type=int, default=8, help="oracle sample size (windows of 49)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


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


def run_reference(a):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    per_step = []
    for _ in range(a.warmup if a.warmup < 1 else 0):
        pass
    for _ in range(a.steps):
        t = oracle_sample_seconds(a.cpu_windows)
        per_step.append(t * WINDOWS / a.cpu_windows)
    t_full = float(np.mean(per_step))
    value = BATCH / t_full
    sample = f"{a.cpu_windows} of 49 CC windows per step (CC+sigma_a+dense partial over them), " \
             f"extrapolated x{WINDOWS / a.cpu_windows:.3g} to one 8192-image batch"
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup,
            "ms_per_step": t_full * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "u64", "data": "synthetic", "impl": "reference",
            "config": {"workload": "C1 Fashion-MNIST-shaped encrypted CNN, CKKS N=2^14 {60,40,40,40,40|60}, "
                                   "batch 8192 in slots", "global_batch": BATCH * a.gpus},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample},
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
    "k_relin_moddown_intt": (490 + 490, 490 + 490),
    "k_relin_moddown_ntt":  (490 + 490, 980 + 490),
}


# Algorithmic HBM bytes per launch (average over the step's launches) of the kernels that
# can dominate: every operand limb read once, every output limb written once (N=2^14).
_LIMB = 8 << 14
C1_ALG_BYTES = {
    # modulus raise: reads (l+1) digit limbs, writes (l+1)^2 raised limbs; l = 3 and 2
    "k_relin_modup": 245 * _LIMB * ((4 + 16) + (3 + 9)) / 2,
    # rescale: reads last limb (2 polys) + kept limbs, writes kept limbs; 4 launches
    "k_rescale_ntt": _LIMB * (245 * 2 * (2 + 4 + 4 + 4) + 245 * 2 * (3 + 3) + 245 * 2 * (2 + 2) + 10 * 2 * 2) / 4,
}


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
    else:
        # C4 (configs[4]) at weak scale: `world` batches of 8192 images, their 49*world
        # (window, batch) units split over the ranks (49 each), dense partials combined by
        # one NCCL uint64 all-reduce, each rank finishing one batch
        sh = parallel.ShardedCNN(ctx, K, kb, W, b, world, rank, world)
        full = []
        for bi in range(world):
            polys = torch.from_numpy(ctx.encode(c1_slots(c1_images(BATCH, 2110 + bi)))).to(f"cuda:{local}")
            full.append(ctx.encrypt_poly(polys, scale=float(2 ** 40), enc_seed=2, obj0=0))
            del polys
        x = parallel.rank_inputs(ctx, sh, full)
        x_sk = None   # rank inputs are gathered ciphertexts: the e2e at N > 1 uses the public-key wire
        del full
        torch.cuda.empty_cache()
        partials = torch.empty(sh.partials_words(), dtype=torch.int64, device=f"cuda:{local}")

        def all_reduce(t):
            dist.all_reduce(t, op=dist.ReduceOp.SUM)   # int64 two's-complement sum == uint64 sum

        def step(inp):
            outs = sh.step(inp, partials, all_reduce)
            return outs[rank]

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(max(a.warmup, 0)):
        step(x)
    stream.synchronize()
    barrier()

    clocks = ClockSampler(local)
    clocks.start()
    l0 = ctx.launches
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    stream.synchronize()
    barrier()
    e0.record(stream)
    for _ in range(a.steps):
        out = step(x)
    e1.record(stream)
    stream.synchronize()
    barrier()
    ms = e0.elapsed_time(e1)
    launches = ctx.launches - l0
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
        copy_stream = torch.cuda.Stream(device=local)
        copied = [torch.cuda.Event() for _ in range(2)]
        used = [torch.cuda.Event() for _ in range(2)]
        trace = [] if os.environ.get("EDL_E2E_TRACE") else None

        def measure_e2e(host_in, unpack_into):
            wire = [torch.empty(host_in.numel(), dtype=torch.int64, device=f"cuda:{local}") for _ in range(2)]

            def run_pipeline(nsteps, first_event=None):
                for k in range(nsteps):
                    buf = k % 2
                    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)] if trace is not None else None
                    with torch.cuda.stream(copy_stream):
                        if k >= 2:
                            copy_stream.wait_event(used[buf])      # step k-2 is done with this buffer
                        if k == 0 and first_event is not None:
                            first_event.record(copy_stream)
                        if ev:
                            ev[0].record(copy_stream)
                        wire[buf].copy_(host_in, non_blocking=True)
                        copied[buf].record(copy_stream)
                        if ev:
                            ev[1].record(copy_stream)
                    stream.wait_event(copied[buf])
                    if ev:
                        ev[2].record(stream)
                    unpack_into(wire[buf], dev_in[buf])
                    res = step(dev_in[buf])
                    host_out[buf].copy_(res.tensor, non_blocking=True)
                    used[buf].record(stream)
                    if ev:
                        ev[3].record(stream)
                        trace.append(ev)

            run_pipeline(2)
            stream.synchronize()
            copy_stream.synchronize()
            barrier()
            f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            if trace is not None:
                trace.clear()
            run_pipeline(a.e2e_steps, first_event=f0)
            f1.record(stream)
            stream.synchronize()
            copy_stream.synchronize()
            barrier()
            if trace:
                t0 = trace[0][0]
                for k, ev in enumerate(trace):
                    print("e2e trace step %d: h2d %.2f-%.2f  compute %.2f-%.2f ms" % (
                        k, t0.elapsed_time(ev[0]), t0.elapsed_time(ev[1]), t0.elapsed_time(ev[2]),
                        t0.elapsed_time(ev[3])), file=sys.stderr)
            te = torch.tensor([f0.elapsed_time(f1)], dtype=torch.float64, device=f"cuda:{local}")
            if world > 1:
                dist.all_reduce(te, op=dist.ReduceOp.MAX)
            del wire
            return world * BATCH * a.e2e_steps / (float(te.item()) / 1e3)

        def pinned(t):
            h = torch.empty(t.numel(), dtype=torch.int64, pin_memory=True)
            h.copy_(t.cpu())
            return h

        # public-key ciphertexts in the packed wire format (edl.h: residues in bit-length-of-q bits)
        host_pk = pinned(ctx.pack(x))
        v_pk = measure_e2e(host_pk, lambda w, o: ctx.unpack(w, x.count, x.level, x.scale, x.key_id, out=o))
        e2e_pk = {"value": v_pk, "unit": UNIT, "h2d_bytes_per_step": int(host_pk.numel() * 8),
                  "d2h_bytes_per_step": int(out_words * 8),
                  "inputs": "public-key ciphertexts, packed wire format (edl_cts_pack/unpack)"}
        del host_pk
        pipeline = ("H2D of step k+1 on a copy stream overlaps step k (2 device input buffers); unpack and "
                    "the step's kernels inside the timed region; 10 output ciphertexts read back every step")
        if x_sk is not None:
            # secret-key ciphertexts of the same images (reading Z16): c0 packed, c1 regenerated on the
            # device from (enc_seed, object id) by edl_cts_unpack_seeded inside each step
            host_sk = pinned(ctx.pack_c0(x_sk))
            v_sk = measure_e2e(host_sk, lambda w, o: ctx.unpack_seeded(w, x_sk.count, x_sk.level, x_sk.scale,
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

    # ---- roofline of the dominant kernel (largest share of the timed region)
    n = ctx.n
    dom = max(prof.items(), key=lambda kv: kv[1][0]) if prof else ("none", (0.0, 0))
    peak_int = ctx.bfly_peak(0)          # q0 (60-bit): Shoup path
    peak_fp = ctx.bfly_peak(1)           # q1 (40-bit): FP64-pipe path
    ntt_roofs = {}
    for name in C1_TRANSFORMS:
        if name in prof and world == 1:
            ach, pk = ntt_roofline(name, prof[name][0], a.steps, n, peak_int, peak_fp)
            ntt_roofs[name] = {"achieved_Gbfly_s": ach / 1e9, "peak_Gbfly_s": pk / 1e9, "frac": ach / pk,
                               "share_of_step": prof[name][0] / ms_instr}
    ntt_doms = [k for k in sorted(prof, key=lambda k: -prof[k][0]) if k in ntt_roofs]
    roof = None
    if ntt_doms:
        k = ntt_doms[0]
        r = ntt_roofs[k]
        traffic = None
        tf = os.path.join(ROOT, "profiles", "round1", "ncu_traffic.json")
        if os.path.exists(tf):
            tj = json.load(open(tf))
            if k in tj:
                traffic = tj[k]["dram_bytes_per_launch"]
        roof = {"kernel": k, "bound": "alu", "unit": "Gbutterfly/s", "achieved": r["achieved_Gbfly_s"],
                "peak": r["peak_Gbfly_s"], "frac": r["frac"], "traffic": traffic,
                "traffic_unit": "DRAM bytes per launch (profiles/round1/ncu_traffic.json, ncu --set full)",
                "algorithmic_bytes_per_launch": C1_ALG_BYTES.get(k),
                "peak_kind": "measured: register-only Harvey CT butterflies (edl_bfly_peak) through the "
                             "kernel's own arithmetic paths, weighted by its 60-bit/40-bit transform mix",
                "peak_int_Gbfly_s": peak_int / 1e9, "peak_fp_Gbfly_s": peak_fp / 1e9,
                "share_of_step": r["share_of_step"], "avg_launch_ms": prof[k][0] / prof[k][1],
                "largest_kernel_overall": dom[0], "all_ntt_kernels": ntt_roofs}
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

    props = torch.cuda.get_device_properties(local)
    device = {"name": props.name, "sms": props.multi_processor_count,
              "smem_per_sm_bytes": getattr(props, "shared_memory_per_multiprocessor", None),
              "l2_bytes": getattr(props, "L2_cache_size", None), "hbm_bytes": props.total_memory}

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        ts = oracle_sample_seconds(a.cpu_windows)
        v = BATCH / (ts * WINDOWS / a.cpu_windows)
        cpu = {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle",
               "sample": f"{a.cpu_windows} of 49 CC windows of one 8192-image batch, extrapolated x"
                         f"{WINDOWS / a.cpu_windows:.3g}"}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
                "warmup": a.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "u64", "data": "synthetic",
                "config": {"workload": ("C1 Fashion-MNIST-shaped encrypted CNN, CKKS N=2^14 {60,40,40,40,40|60}, "
                                        "batch 8192 in slots (784 pixel ciphertexts), CC 5x4x4/4 -> sigma_a -> "
                                        "dense 245->10") if world == 1 else
                                       (f"C4 scale-out CNN: {world} batches of 8192 synthetic images (C1 "
                                        f"architecture and parameters), 49*{world} (window, batch) units over "
                                        f"{world} GPUs"), "global_batch": BATCH * world,
                           "parallelism": ("single GPU" if world == 1 else
                                           f"C4 (window, batch) units sharded x{world}, NCCL uint64 all-reduce of "
                                           f"dense partials"),
                           "l2": "inputs 1.03 GB per GPU > L2 (no flush)"},
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
                "clocks": clk, "dominant_kernel": dom[0], "kernels": kernels, "device": device,
                "kernel_timing": {"method": "CUDA event pair around every launch, on the library stream, over a "
                                            "second pass of the same K steps", "ms_per_step_instrumented":
                                  ms_instr / a.steps},
                "replica_dp": replica,
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
