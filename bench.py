#!/usr/bin/env python3
"""Optimizer-update throughput on B200: params updated / s (BASELINE.json metric).

Workload (BASELINE.json configs[1]): all six optimizers -- AdamW, Lion, Adan,
Sophia, LOMO, AdaLomo -- each updating a LLaMA-7B-shaped synthetic parameter set
(291 tensors, 6,738,415,616 fp32 params, registry order) once per step.  LOMO and
AdaLomo include the global gradient-norm clipping pass (north_star; clip = 1.0):
LOMO = deterministic Σg² pass + clipped update (16 B/param), AdaLomo = clip fused
into its first pass (24 B/param).  One "step" = one update of the whole set by each
of the six optimizers in turn; value = 6 * P * K / (device time of the K timed
steps).  Inputs are synthetic (counter-based generator), fp32, resident in HBM,
27 GB per buffer (> L2), so no L2 flush is needed between iterations.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

--gpus N > 1 without a torchrun environment re-launches itself under
torch.distributed.run with N local ranks (one process per GPU, NCCL); under torchrun
WORLD_SIZE must equal N.  At N > 1 each optimizer runs the WHOLE data-parallel step
of the reference's stage-2 branch (parallel.cpp:656-666) on the same 7B set
(strong scaling): every rank holds its local gradients for all P params,
    stored-state kinds  reduce-scatter(SUM, fp32 grads) -> fused update of the
                        ZeroPlan-owned slice -> all-gather(fp32 params)
    LOMO + clip         reduce-scatter -> Σg² of the owned slice -> all-reduce(1 fp64)
                        -> clipped update -> all-gather
    AdaLomo + clip      row-split: reduce-scatter (rank-major layout) -> pass 1 ->
                        all-reduce(column sums, Σg², Σp², Σv_row) -> pass 2 ->
                        all-reduce(Σu²) -> pass 3 -> all-gather
value = 6 * P / Σ max-over-ranks step time.  Beside it: the shard-local update time
(the same kernels without the collectives), the NVLink bytes per rank, and the
measured NCCL bus bandwidth they are bounded by.

e2e: the same metric through the public API with HOST (pinned) buffers -- per step
H2D params+grads, the update, D2H params (C-ABI host-span calls).  cpu_baseline /
--impl reference: the reference's own minicollie::optim (oracle/_ref, compiled from
its sources, driven through oracle/oracle.py only -- no product code) on this host's
cores on a bounded registry-order sample (5 decoder layers of the 7B set: 45 tensors,
1.01e9 params, fewer layers when host RAM is short).
"""
from __future__ import annotations

import argparse
import gc
import json
import math
import os
import socket
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

KINDS = ["adamw", "lion", "adan", "sophia", "lomo", "adalomo"]
STORED = ("adamw", "lion", "adan", "sophia")
CLIP = 1.0  # LOMO / AdaLomo global grad-norm clip threshold (optim.cpp:291-303)
# Algorithmic (dependency-forced) HBM bytes per parameter, fp32:
# LOMO with its clip pass 16 (Σg² pass reads g; update reads p, g, writes p),
# AdaLomo with the clip fused into pass 1 24.
BYTES_PER_PARAM = {"adamw": 28, "lion": 20, "adan": 44, "sophia": 24, "lomo": 16,
                   "adalomo": 24}
# Paper Table 4 hyper-parameters for throughput runs; Sophia: defaults.
HPARAMS = {"adamw": dict(lr=1e-5, weight_decay=1e-2), "lion": dict(lr=3e-6, weight_decay=3e-2),
           "adan": dict(lr=5e-5, weight_decay=2e-2), "sophia": dict(lr=1e-4),
           "lomo": dict(lr=1e-2), "adalomo": dict(lr=5e-4)}
NVLINK_NOMINAL_GBS = 900.0  # NVLink 5, per direction per GPU


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._th = None

    def start(self):
        def run():
            while not self._stop.is_set():
                try:
                    out = subprocess.run(
                        ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                         "--format=csv,noheader,nounits"], capture_output=True, text=True,
                        timeout=10).stdout.strip()
                    if out:
                        self.rows.append([x.strip() for x in out.split(",")])
                except Exception:
                    pass
                self._stop.wait(0.2)

        self._th = threading.Thread(target=run, daemon=True)
        self._th.start()

    def stop(self):
        self._stop.set()
        if self._th:
            self._th.join(timeout=15)

    def summary(self):
        import statistics

        sm = [float(r[1]) for r in self.rows if len(r) > 2 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) > 2 and r[2].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            for k, nm in enumerate(names):
                if len(r) > 5 + k and r[5 + k].lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(self.rows)}


# ---------------------------------------------------------------------------------------
# reference arm / CPU baseline: the reference's own code on the host cores.  Only
# oracle/ is imported here (the compiled reference + its kind parser and defaults).
# ---------------------------------------------------------------------------------------

def _oracle():
    p = os.path.join(ROOT, "oracle")
    if p not in sys.path:
        sys.path.insert(0, p)
    import oracle as O

    if O.ref is None:
        raise RuntimeError("oracle/_ref/libmco_ref.so missing (run __graft_entry__.build())")
    return O


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def host_available_bytes() -> int:
    try:
        with open("/proc/meminfo") as f:
            for ln in f:
                if ln.startswith("MemAvailable:"):
                    return int(ln.split()[1]) * 1024
    except Exception:
        pass
    return 16 << 30


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def cpu_sample_shapes(O):
    """Registry-order run of whole decoder layers of the 7B set (tensors 1..9L): the
    reference spreads LOMO / AdaLomo over tensors, so the sample holds more tensors
    than host threads; 5 layers = 45 tensors, 1,011,916,800 params (a
    1e9-param 7B sample), fewer layers if the host cannot hold Adan's 48 B/param fp64
    working set in half its free RAM."""
    if os.environ.get("MCO_CPU_SAMPLE") == "tiny":  # CPU test of the bench contract
        return O.llama_shapes(256, 688, 8, 8192)[1:19], 2
    per_layer = 4 * 4096 * 4096 + 3 * 4096 * 11008 + 2 * 4096
    layers = int(max(1, min(5, host_available_bytes() * 0.5 // (48 * per_layer))))
    return O.llama_shapes(4096, 11008, 32, 32000)[1:1 + 9 * layers], layers


def run_cpu_reference(warmup: int, steps: int):
    O = _oracle()
    shapes, layers = cpu_sample_shapes(O)
    n = sum(math.prod(s) for s in shapes)
    threads = host_threads()
    per, total = {}, 0.0
    for k in KINDS:
        cfg = O.ref_config(k, **HPARAMS[k])
        clip = CLIP if k in ("lomo", "adalomo") else None
        sec = O.ref_bench(cfg, shapes, threads, warmup, steps, clip=clip)
        per[k] = {"ms": round(sec * 1e3, 2), "params_per_s": n / sec}
        total += sec
        log(f"[cpu-ref] {k}: {sec * 1e3:.1f} ms/step, {n / sec / 1e9:.3f} Gparam/s "
            f"({threads} threads)")
    value = len(KINDS) * n / total
    sample = (f"{layers} registry-order decoder layers of the 7B set ({len(shapes)} tensors, "
              f"{n} fp64 params) per optimizer, {warmup} warm-up + {steps} timed steps; "
              "stored-state kinds: one FlatOptimizer per thread over disjoint slices; "
              "LOMO / AdaLomo: tensors spread largest-first over the threads, with the "
              f"global grad-norm clip pass (clip {CLIP})")
    return value, threads, sample, per, total / max(steps, 1), n


def run_cpu_single_thread():
    """The reference on ONE host thread (T = nproc and T = 1): the first
    q-projection matrix of the 7B registry."""
    O = _oracle()
    shapes = [(4096, 4096)]
    n = 4096 * 4096
    per, total = {}, 0.0
    for k in KINDS:
        clip = CLIP if k in ("lomo", "adalomo") else None
        sec = O.ref_bench(O.ref_config(k, **HPARAMS[k]), shapes, 1, 1, 1, clip=clip)
        per[k] = {"ms": round(sec * 1e3, 2), "params_per_s": n / sec}
        total += sec
    return {"value": len(KINDS) * n / total, "unit": "params/s", "cores": 1,
            "sample": f"one 4096x4096 matrix ({n} fp64 params) per optimizer, 1 warm-up + "
                      "1 timed step", "per_optimizer": per}


# ---------------------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------------------

def make_cfg(kind: str):
    from paper_2312_00407_b200.optim import OptimizerConfig, parse_kind

    cfg = OptimizerConfig.defaults_for(parse_kind(kind))
    for a, v in HPARAMS[kind].items():
        setattr(cfg, a, v)
    return cfg


class Stepper:
    """One optimizer over the flat registry buffers through the public API.

    world == 1: the whole set on this GPU.  world > 1: the whole data-parallel step
    (module docstring), and `local()` = the same update kernels on this rank's part
    without the collectives (the shard-local figure)."""

    def __init__(self, kind, shapes, P, bp, bg, world, rank, comm=None, bucket=0):
        from paper_2312_00407_b200 import optim, zero

        self.kind, self.world, self.rank = kind, world, rank
        self.cfg = make_cfg(kind)
        self.lr = self.cfg.lr
        self.P = P
        self.p, self.g = bp[:P], bg[:P]
        self.n_local = P
        dev = bp.device.index
        if world == 1:
            if kind in STORED:
                self.opt = optim.FlatOptimizer(self.cfg, P, device=dev)
                self._step = lambda: self.opt.step(self.p, self.g, self.lr)
            elif kind == "lomo":
                self._norm = None

                def lomo():
                    self._norm = optim.lomo_step(self.p, self.g, self.lr, clip=CLIP)
                self._step = lomo
            else:
                self.opt = optim.AdaLomoState(self.cfg, shapes, device=dev, grad_clip=CLIP)
                self._step = lambda: self.opt.apply_all(self.p, self.g, self.lr)
            self.local = self._step
            return
        plan = zero.ZeroPlan.make(P, world, 2)
        lo, hi = plan.owned_range(rank)
        self.n_local = hi - lo
        if kind in STORED:
            if comm is not None:  # NCCL: the C-ABI bucketed, double-buffered step (mco_zb)
                self.opt = zero.BucketedZeroOptimizer(self.cfg, P, comm, bucket_elems=bucket)
                self._step = lambda: self.opt.step(self.p, self.g, self.lr)
                self.local = lambda: self.opt.step_local(self.p, self.g, self.lr)
                self.n_local = self.opt.owned
            else:  # gloo (several ranks on one GPU in the tests): torch.distributed
                self.opt = zero.ZeroShardedOptimizer(self.cfg, P, device=dev)
                flat = self.opt.opt
                self._step = lambda: self.opt.step(self.p, self.g, self.lr)
                po, go = self.p[lo:hi], self.g[lo:hi]
                self.local = lambda: flat.step(po, go, self.lr)
        elif kind == "lomo":
            self.opt = zero.ZeroShardedLomo(P, CLIP)
            self._step = lambda: self.opt.step(self.p, self.g, self.lr)
            po, go = self.p[lo:hi], self.g[lo:hi]
            self.local = lambda: zero.sharded_lomo_step(po, go, self.lr, CLIP)
        else:
            self.rs = zero.RowShardedAdaLomo(self.cfg, shapes, device=dev, grad_clip=CLIP)
            L = world * self.rs.chunk
            if L > bp.numel():
                raise RuntimeError(f"rank-major AdaLomo buffers need {L} elements")
            self.p, self.g = bp[:L], bg[:L]
            self.n_local = self.rs.local_numel
            c = self.rs.chunk
            lp = self.p[rank * c:rank * c + self.n_local]
            lg = self.g[rank * c:rank * c + self.n_local]
            self._step = lambda: self.rs.step_dp(self.p, self.g, self.lr)
            self.local = lambda: self.rs.step(lp, lg, self.lr)

    def step(self):
        self._step()

    def steps_taken(self):
        o = getattr(self, "opt", None)
        if o is not None and not hasattr(o, "steps_taken"):
            o = getattr(o, "opt", None)  # ZeroShardedOptimizer keeps its FlatOptimizer in .opt
        return o.steps_taken() if hasattr(o, "steps_taken") else 0


def nvlink_bytes_per_rank(kind, P, world, rs_chunk=None, payload=0):
    """Bytes each rank sends (= receives) per step over NVLink in the ring collectives:
    reduce-scatter + all-gather of fp32 move (N-1)/N of the buffer each; the scalar /
    payload all-reduces move 2 (N-1)/N of theirs."""
    f = (world - 1) / world
    if kind == "adalomo":
        L = world * rs_chunk
        return int(f * L * 4 * 2 + 2 * f * payload * 8)
    return int(f * P * 4 * 2 + (2 * f * 8 if kind == "lomo" else 0))


def nccl_busbw(dev, world, nbytes=1 << 30):
    """Measured all-gather bus bandwidth (GB/s per rank and direction) over this job's
    NCCL communicator: (N-1)/N * bytes / time, best of 3."""
    import torch
    import torch.distributed as dist

    n = nbytes // 4 // world * world
    out = torch.empty(n, device=dev)
    inp = out[:n // world].clone()
    best = 0.0
    for _ in range(4):
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        dist.all_gather_into_tensor(out, inp)
        e1.record()
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) * 1e-3], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        best = max(best, (world - 1) / world * n * 4 / t.item() / 1e9)
    del out, inp
    return round(best, 1)


def timed_block(fn, steps, stream, per_step=False):
    import torch

    evs = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
    evs[0].record(stream)
    for i in range(steps):
        fn()
        evs[i + 1].record(stream)
    torch.cuda.synchronize()
    ms = evs[0].elapsed_time(evs[-1]) / steps
    return (ms, [evs[i].elapsed_time(evs[i + 1]) for i in range(steps)]) if per_step else ms


def bench_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_2312_00407_b200 import optim, registry, zero

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    model = registry.MODELS[args.model]
    if args.layers:
        model = registry.layer_subset(model, args.layers)
    shapes = model.shapes()
    P = model.param_count()
    kinds = args.optimizers.split(",")
    hbm_peak, peak_src = measured_peaks()
    backend = dist.get_backend() if world > 1 else None
    log(f"[rank {rank}] model {model.name} P={P} world={world} kinds={kinds}")

    # one pair of flat buffers for every kind (rank-major AdaLomo needs a little more)
    cap = P
    if world > 1 and "adalomo" in kinds:
        probe = zero.RowShardedAdaLomo.chunk_len(shapes, world)
        cap = max(P, world * probe)
    bp = torch.empty(cap, dtype=torch.float32, device=dev)
    bg = torch.empty(cap, dtype=torch.float32, device=dev)
    registry.fill_params(bp[:P], shapes)
    registry.fill_grads(bg[:P], shapes, 1)
    if cap > P:
        bp[P:].zero_()
        bg[P:].zero_()
    torch.cuda.synchronize()
    comm = None
    busbw = None
    if world > 1:
        if backend == "nccl":
            comm = zero.NcclComm(device=local_rank)
            busbw = nccl_busbw(dev, world)
            log(f"[rank {rank}] NCCL all-gather bus bandwidth {busbw} GB/s")

    stream = torch.cuda.current_stream()
    per, total_ms, launches = {}, 0.0, 0
    clocks = ClockSampler(local_rank)
    for kind in kinds:
        st = Stepper(kind, shapes, P, bp, bg, world, rank, comm, args.bucket_elems)
        for _ in range(args.warmup):
            st.step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        l0 = optim.launch_count()
        if kind == kinds[0]:
            clocks.start()
        t0 = st.steps_taken()
        ms, step_ms = timed_block(st.step, args.steps, stream, per_step=True)
        launches_kind = optim.launch_count() - l0
        launches += launches_kind
        rep_ms = [ms] + [timed_block(st.step, args.steps, stream)
                         for _ in range(max(args.repeats, 1) - 1)]
        local_ms = None
        if world > 1:
            torch.cuda.synchronize()
            dist.barrier()
            local_ms = timed_block(st.local, args.steps, stream)
            t = torch.tensor([ms, local_ms], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms, local_ms = t.tolist()
        bpp = BYTES_PER_PARAM[kind]
        gbs = bpp * st.n_local / (ms * 1e-3) / 1e9  # per GPU (this rank's update bytes)
        e = {"ms": round(ms, 4), "params_per_s": P / (ms * 1e-3), "bytes_per_param": bpp,
             "achieved_gbs_per_gpu": round(gbs, 1),
             "frac_of_measured_hbm": round(gbs / hbm_peak, 4),
             "params_per_launch": st.n_local,
             "launches_per_step": args.steps and (launches_kind / args.steps),
             "repeats": len(rep_ms),
             "ms_median_of_repeats": round(sorted(rep_ms)[len(rep_ms) // 2], 4),
             "ms_min_max_of_repeats": [round(min(rep_ms), 4), round(max(rep_ms), 4)]}
        if kind in ("lomo", "adalomo"):
            e["clip"] = CLIP
        if world > 1:
            lgbs = bpp * st.n_local / (local_ms * 1e-3) / 1e9
            payload = 0
            if kind == "adalomo":
                payload = sum(t.numel() for t in (st.rs.state.payload(0), st.rs.state.payload(1)))
            nvb = nvlink_bytes_per_rank(kind, P, world, getattr(getattr(st, "rs", None),
                                                                "chunk", None), payload)
            e["shard_local"] = {
                "ms": round(local_ms, 4), "params_per_s": P / (local_ms * 1e-3),
                "frac_of_measured_hbm": round(lgbs / hbm_peak, 4),
                "what": "the same update kernels on this rank's part, no gradient "
                        "reduce-scatter / parameter all-gather (max over ranks)"}
            e["nvlink"] = {"bytes_per_rank_per_direction": nvb,
                           "gb_per_s": round(nvb / (ms * 1e-3) / 1e9, 1),
                           "frac_of_nominal": round(nvb / (ms * 1e-3) / 1e9
                                                    / NVLINK_NOMINAL_GBS, 4)}
            if busbw:
                e["nvlink"]["frac_of_measured_busbw"] = round(
                    nvb / (ms * 1e-3) / 1e9 / busbw, 4)
            # the step cannot beat max(collective bytes / bus bw, update bytes / HBM)
            if busbw:
                e["roofline_ms"] = round(max(nvb / (busbw * 1e9), bpp * st.n_local
                                             / (hbm_peak * 1e9)) * 1e3, 3)
        if kind == "sophia":
            k = st.cfg.update_interval
            ref = [m for i, m in enumerate(step_ms) if (t0 + i) % k == 0]  # t-1 = t0+i
            non = [m for i, m in enumerate(step_ms) if (t0 + i) % k != 0]
            for name, xs, b in (("refresh", ref, 28), ("non_refresh", non, 24)):
                if xs:
                    m = sum(xs) / len(xs)
                    e[name] = {"steps": len(xs), "ms": round(m, 4), "bytes_per_param": b,
                               "frac_of_measured_hbm": round(
                                   b * st.n_local / (m * 1e-3) / 1e9 / hbm_peak, 4)}
        per[kind] = e
        total_ms += ms
        log(f"[rank {rank}] {kind}: {ms:.3f} ms/step, {P / ms / 1e6:.1f} Gparam/s (all GPUs), "
            f"{gbs:.0f} GB/s/GPU = {gbs / hbm_peak:.3f} of {peak_src} HBM"
            + (f"; shard-local {local_ms:.3f} ms" if local_ms else ""))
        del st
        gc.collect()
        torch.cuda.synchronize()
    clocks.stop()
    value = len(per) * P / (total_ms * 1e-3)
    extra = {}
    if world == 1 and "sophia" in per and not args.no_extra:
        # Sophia precise-m (state "f32m64": fp64 m, the per-element 1e-5 bar met); not
        # part of `value` -- the six-kind step uses the fp32 product path
        cfg = make_cfg("sophia")
        opt = optim.FlatOptimizer(cfg, P, state_dtype="f32m64")
        pp, gg = bp[:P], bg[:P]
        for _ in range(args.warmup):
            opt.step(pp, gg, cfg.lr)
        ms = timed_block(lambda: opt.step(pp, gg, cfg.lr), args.steps, stream)
        gbs = 32 * P / (ms * 1e-3) / 1e9
        extra["sophia_precise_m"] = {
            "ms": round(ms, 4), "params_per_s": P / (ms * 1e-3), "bytes_per_param": 32,
            "frac_of_measured_hbm": round(gbs / hbm_peak, 4),
            "what": "Sophia with an fp64 first moment (state f32m64, sophia_m64_tma); "
                    "refresh steps write h too (+4 B)", "parity": load_parity("sophia_m64")}
        per["sophia"]["parity_fp32_m"] = load_parity("sophia")
        del opt
        gc.collect()
        log(f"[rank {rank}] sophia precise-m: {ms:.3f} ms/step, {gbs / hbm_peak:.3f} of HBM")

    # dominant kernel = the optimizer with the largest share of the step (N = 1)
    dom = max(per, key=lambda k: per[k]["ms"] if world == 1 else
              per[k]["shard_local"]["ms"])
    src = per[dom] if world == 1 else per[dom]["shard_local"]
    npl = per[dom]["params_per_launch"]
    achieved = BYTES_PER_PARAM[dom] * npl / (src["ms"] * 1e-3) / 1e9
    kname = {"lomo": "sumsq_kernel + lomo_tma_kernel (clip)",
             "adalomo": "k1_stats .. k6_update (clip fused into pass 1)"}.get(
        dom, "flat_tma_kernel: cp.async.bulk + mbarrier pipeline"
        if optim.flat_variant() == "tma" else f"flat_step_kernel, variant {optim.flat_variant()}")
    roofline = {"bound": "hbm", "kernel": f"{dom} update ({kname})",
                "achieved": round(achieved, 1), "peak": hbm_peak, "peak_source": peak_src,
                "unit": "GB/s", "frac": round(achieved / hbm_peak, 4),
                "algorithmic_bytes_per_param": BYTES_PER_PARAM[dom], "params_per_launch": npl,
                "traffic": load_traffic(dom, npl)}
    if world > 1:
        roofline["note"] = ("dominant shard-local update kernel; the whole step at N > 1 is "
                            "bounded by the collectives (per_optimizer.*.nvlink)")
    out = dict(value=value, ms_per_step=total_ms, per=per, roofline=roofline, extra=extra,
               launches=launches, clocks=clocks.summary(), P=P, owned=P, shapes=shapes,
               kinds=[k for k in kinds if k in per], p=bp[:P], g=bg[:P], dev=dev,
               busbw=busbw)
    if world > 1:
        out["lo"], hi = zero.ZeroPlan.make(P, world, 2).owned_range(rank)
        out["owned"] = hi - out["lo"]
    if world > 1 and not args.no_e2e:
        try:  # every rank takes part (max-over-ranks time); failures are reported
            out["e2e"] = bench_e2e(args, out, rank, world)
        except Exception as ex:
            log(f"[rank {rank}] e2e failed: {ex!r}")
            out["e2e"] = None
    return out


C4_BYTES = {"adan": 46, "sophia": 26, "adamw": 30, "lion": 22}  # mixed, SURVEY 8(d)


def bench_c4(args, rank, world, local_rank):
    """BASELINE configs[3]: ZeRO stage-2 Adan / Sophia on a LLaMA-65B-
    shaped set over the bucketed, double-buffered C-ABI step (mco_zb): fp32 master +
    state of each rank's pieces, bf16 replicas (ring mode -- buckets gathered into two
    slots, the stage-3 layout -- when the full replicas do not fit), fp32 gradients
    arriving bucket by bucket into the library's two staging slots (no full-length
    gradient is resident; the backward that would produce them is not timed, the
    staged values are reused).  Per step and bucket: reduce-scatter (fp32) -> update ->
    all-gather (bf16), RS(k+1) overlapping update(k).  One JSON line per kind."""
    import torch
    import torch.distributed as dist

    from paper_2312_00407_b200 import optim, registry, zero

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    model = registry.MODELS[args.model]
    if args.layers:
        model = registry.layer_subset(model, args.layers)
    P = model.param_count()
    hbm_peak, peak_src = measured_peaks()
    comm = zero.NcclComm(device=local_rank)
    busbw = nccl_busbw(dev, world) if world > 1 else None
    stream = torch.cuda.current_stream()
    kinds = [k for k in args.optimizers.split(",") if k in STORED]
    for kind in kinds:
        cfg = make_cfg(kind)
        gc.collect()
        torch.cuda.empty_cache()
        free = torch.cuda.mem_get_info()[0]
        fp = zero.BucketedZeroOptimizer.footprint(int(cfg.kind), P, world, args.bucket_elems, 2)
        ring = fp["total"] > free * 0.97
        if ring:
            fp = zero.BucketedZeroOptimizer.footprint(int(cfg.kind), P, world,
                                                      args.bucket_elems, 2, True)
        zb = zero.BucketedZeroOptimizer(cfg, P, comm, bucket_elems=args.bucket_elems,
                                        replica_dtype=torch.bfloat16)
        optim.synth_fill(zb.master(), registry.SEED, 0, 0xFFFB, 0, 0, -6)
        rep = None if ring else torch.zeros(P, dtype=torch.bfloat16, device=dev)
        for k in (0, 1):
            if k < zb.nbuckets:
                optim.synth_fill(zb.grad_buffer(k), registry.SEED, 1, 0xFFFB, 1, 0, -7, 10)

        def one():
            zb.begin(rep, cfg.lr)
            for k in reversed(range(zb.nbuckets)):
                zb.grad_buffer(k)  # the slot is free (its previous bucket was reduced)
                zb.grad_ready(k)
            zb.end()

        for _ in range(args.warmup):
            one()
        comm.wait()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        ms = timed_block(one, args.steps, stream)
        comm.check()
        if world > 1:
            t = torch.tensor([ms], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = t.item()
        f = (world - 1) / world
        nvb = int(f * P * 4 + f * P * 2)  # RS fp32 grads + AG bf16 params, per direction
        hbm_b = C4_BYTES[kind] * zb.owned
        line = {"metric": f"C4 ZeRO stage-2 {kind} step (params/s, whole job)",
                "value": P / (ms * 1e-3), "unit": "params/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
                "higher_is_better": True, "scaling": "strong", "dtype": "f32 master/state, "
                "bf16 replicas, f32 grads", "data": "synthetic",
                "config": {"workload": "configs[3]", "model_shape": model.name, "params": P,
                           "bucket_elems": zb.bucket_elems, "buckets": zb.nbuckets,
                           "mode": "ring (stage-3 layout)" if ring else "bf16 replicas",
                           "per_rank_bytes": fp},
                "hbm": {"update_bytes_per_rank": hbm_b, "peak": hbm_peak,
                        "peak_source": peak_src,
                        "bound_ms": round(hbm_b / (hbm_peak * 1e9) * 1e3, 3)},
                "nvlink": {"bytes_per_rank_per_direction": nvb,
                           "gb_per_s": round(nvb / (ms * 1e-3) / 1e9, 1),
                           "nominal_gbs": NVLINK_NOMINAL_GBS, "measured_busbw_gbs": busbw,
                           "bound_ms": round(nvb / ((busbw or NVLINK_NOMINAL_GBS) * 1e9)
                                             * 1e3, 3)}}
        line["roofline_ms"] = max(line["hbm"]["bound_ms"], line["nvlink"]["bound_ms"])
        line["frac"] = round(line["roofline_ms"] / ms, 4)
        if rank == 0:
            print(json.dumps(line), flush=True)
            log(f"[c4] {kind}: {ms:.2f} ms/step, {P / ms / 1e6:.1f} Gparam/s, roofline "
                f"{line['roofline_ms']:.2f} ms ({'ring' if ring else 'replicas'})")
        del zb, rep
    comm.wait()


def load_parity(kind):
    """Measured fp32-vs-fp64-reference errors of `kind` (profiles/parity.json, written by
    tests/test_gpu_flat.py on the GPU: fraction of elements past 1e-5 and the largest
    error) -- bench.py never runs the oracle itself."""
    try:
        with open(os.path.join(ROOT, "profiles", "parity.json")) as f:
            return json.load(f).get(kind)
    except Exception:
        return None


def load_traffic(kind, params_per_launch):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch, from the committed
    ncu --set full capture (profiles/traffic.json holds DRAM bytes per parameter per
    step measured on a layer subset of the same shapes), scaled to this launch."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            d = json.load(f)[kind]
        return round(d["dram_bytes_per_param"] * params_per_launch)
    except Exception:
        return None


def pcie_ceiling(hp, dev):
    """Pinned-host copy bandwidth on this box (GB/s): H2D, D2H, and both at once
    (two streams) -- the roofline of the host-buffer path."""
    import torch

    n = min(hp.numel(), 1 << 28)  # 1 GiB
    d = torch.empty(n, device=dev)
    d2 = torch.empty(n, device=dev)
    h2 = torch.empty(n, dtype=torch.float32, pin_memory=True)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def bw(fn, nbytes, it=4):
        fn()
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(it):
            fn()
        torch.cuda.synchronize()
        return nbytes * it / (time.perf_counter() - t) / 1e9

    def both():
        with torch.cuda.stream(s1):
            d.copy_(hp[:n], non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)

    out = {"h2d_gbs": bw(lambda: d.copy_(hp[:n], non_blocking=True), 4 * n),
           "d2h_gbs": bw(lambda: h2.copy_(d, non_blocking=True), 4 * n),
           "both_gbs": bw(both, 8 * n)}
    del d, d2, h2
    return {k: round(v, 1) for k, v in out.items()}


def bench_e2e(args, res, rank=0, world=1):
    """Host-buffer end-to-end: per step H2D(p, g) + update + D2H(p) through the C-ABI
    host-span calls (LOMO / AdaLomo with their clip).  N > 1: every rank runs its own
    part (the ZeroPlan slice for the flat kinds and LOMO, every N-th tensor for AdaLomo)
    over its own PCIe link; per-kind time = max over ranks; bytes are whole-job."""
    import torch

    from paper_2312_00407_b200 import optim

    def max_over_ranks(x):
        if world == 1:
            return x
        import torch.distributed as dist

        t = torch.tensor([x], dtype=torch.float64, device=res["dev"])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.item()

    def barrier():
        if world > 1:
            import torch.distributed as dist

            dist.barrier()

    P = res["owned"]
    shapes = res["shapes"] if world == 1 else res["shapes"][rank::world]
    n_ada = sum(math.prod(s) for s in shapes)
    need = 2 * max(P, n_ada) * 4 * 1.3
    avail = host_available_bytes() / world
    fits = need < avail * 0.6
    n = P
    if world == 1 and not fits:  # whole tensors prefix that fits
        cap = int(avail * 0.6 / (2 * 4 * 1.3)) // 1024 * 1024
        acc, k = 0, 0
        while k < len(shapes) and acc + math.prod(shapes[k]) <= cap:
            acc += math.prod(shapes[k])
            k += 1
        shapes, n = shapes[:k], acc
        n_ada = n
    ok = 1.0 if (world == 1 or fits) else 0.0
    if world > 1:  # every rank takes the same branch (collectives follow)
        ok = -max_over_ranks(-ok)
    if ok < 1.0:
        raise RuntimeError(f"e2e: host memory for {max(P, n_ada)} params per rank unavailable "
                           f"on some rank (this rank: {avail / 1e9:.1f} GB available share)")
    log(f"[e2e] rank {rank}: host buffers {n} params ({'full part' if n == P else 'prefix'}), "
        f"AdaLomo {len(shapes)} tensors / {n_ada} params, pinned")
    m = max(n, n_ada)
    hp = torch.empty(m, dtype=torch.float32, pin_memory=True)
    hg = torch.empty(m, dtype=torch.float32, pin_memory=True)
    lo = res.get("lo", 0)
    src_p, src_g = res["p"][lo:lo + n].cpu(), res["g"][lo:lo + n].cpu()
    for a in range(0, m, n):  # the part's values, repeated when AdaLomo's subset is larger
        b = min(m, a + n)
        hp[a:b].copy_(src_p[:b - a])
        hg[a:b].copy_(src_g[:b - a])
    del src_p, src_g
    dev = res["p"].device
    # the device-timed legs' buffers (54 GB for 7B) are not needed any more: free them, so
    # the host-span calls have the device to themselves (LOMO's clip path keeps the
    # gradient resident when there is room: 8 instead of 12 B/param up)
    res["p"] = res["g"] = None
    gc.collect()
    torch.cuda.empty_cache()
    pcie = pcie_ceiling(hp, dev)
    log(f"[e2e] rank {rank}: PCIe ceiling (pinned, GB/s): {pcie}")
    steps = max(1, min(args.steps, args.e2e_steps))
    tot_s, h2d, d2h, h2d_me, d2h_me, bound_serial = 0.0, 0, 0, 0, 0, 0.0
    per = {}
    opt = ada = one = None
    for kind in res["kinds"]:
        cfg = make_cfg(kind)
        opt = ada = one = None  # free the previous optimizer's device state first
        gc.collect()
        k_n = n_ada if kind == "adalomo" else n
        hpn, hgn = hp[:k_n].numpy(), hg[:k_n].numpy()
        if kind in STORED:
            opt = optim.FlatOptimizer(cfg, k_n)

            def one():
                opt.step(hpn, hgn, cfg.lr)  # mco_flat_step_host: pipelined H2D/step/D2H
        elif kind == "adalomo":
            ada = optim.AdaLomoState(cfg, shapes, grad_clip=CLIP)

            def one():
                ada.apply_all(hpn, hgn, cfg.lr)  # g up + stats, then per tensor p up/update/down
        else:
            def one():
                optim.lomo_step(hpn, hgn, cfg.lr, clip=CLIP)  # mco_lomo_apply_host: g resident
        one()
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        for _ in range(steps):
            one()
        torch.cuda.synchronize()
        dt = max_over_ranks((time.perf_counter() - t0) / steps)
        total = res["P"] if world > 1 else k_n  # params of the whole job this step
        # LOMO / AdaLomo with the clip: no parameter may move before every gradient has
        # arrived, so the gradients go up first (resident on the device: 4 B/param), then
        # the parameters go up and come back down overlapped (full duplex).  LOMO falls
        # back to streaming g twice (12 B/param up) when the device has no room for it.
        hb = 8
        if kind == "lomo" and torch.cuda.mem_get_info()[0] < 4 * k_n + (2 << 30):
            hb = 12
        per[kind] = {"ms": round(dt * 1e3, 2), "params_per_s": total / dt,
                     "h2d_bytes_per_param": hb, "d2h_bytes_per_param": 4}
        tot_s += dt
        h2d += hb * total
        d2h += total * 4
        if kind in ("lomo", "adalomo"):
            gb = (hb - 4) * k_n  # gradient upload(s) before any parameter is final
            bound_serial += gb / (pcie["h2d_gbs"] * 1e9) + max(
                4 * k_n / (pcie["h2d_gbs"] * 1e9), 4 * k_n / (pcie["d2h_gbs"] * 1e9),
                8 * k_n / (pcie["both_gbs"] * 1e9))
        else:
            h2d_me += hb * k_n
            d2h_me += k_n * 4
        if rank == 0:
            log(f"[e2e] {kind}: {dt * 1e3:.1f} ms/step, {total / dt / 1e9:.2f} Gparam/s")
    # the copies bound the step: max(H2D bytes / H2D BW, D2H / D2H BW, all / both-ways BW)
    # over this rank's own link (every rank has one)
    bound_s = max(h2d_me / (pcie["h2d_gbs"] * 1e9), d2h_me / (pcie["d2h_gbs"] * 1e9),
                  (h2d_me + d2h_me) / (pcie["both_gbs"] * 1e9)) + bound_serial
    total_params = res["P"] if world > 1 else n
    return {"value": len(per) * total_params / tot_s, "unit": "params/s",
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "params": total_params,
            "per_optimizer": per,
            "roofline": {"bound": "pcie", "achieved": round((h2d + d2h) / tot_s / 1e9, 1),
                         "unit": "GB/s", "peak": pcie,
                         "peak_source": "measured in this run" + (" (rank 0's link)"
                                                                 if world > 1 else ""),
                         "frac": round(bound_s / tot_s, 4)},
            "path": "C-ABI host-span calls on pinned host buffers: mco_flat_step_host, "
                    "mco_lomo_apply_host and mco_adalomo_apply_all_host (with the clip: "
                    "H2D g + its statistics, then H2D p / update / D2H p overlapped)" + (
                        f"; each of {world} ranks over its own part" if world > 1 else "")}


def free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def relaunch(n: int) -> int:
    """`python bench.py --gpus N` outside torchrun: run this script under
    torch.distributed.run with N local ranks (rank 0 prints the line)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={n}", "--master-addr", "127.0.0.1",
           "--master-port", str(free_port()), os.path.abspath(__file__), *sys.argv[1:]]
    log(f"[bench] --gpus {n}: launching {n} ranks: {' '.join(cmd[1:6])} ...")
    return subprocess.run(cmd).returncode


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--model", default="llama-7b")
    ap.add_argument("--layers", type=int, default=0,
                    help="decoder-layer subset of --model (profiling runs only)")
    ap.add_argument("--optimizers", default=",".join(KINDS))
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra", action="store_true",
                    help="skip the legs reported beside the value (Sophia precise-m)")
    ap.add_argument("--cpu-steps", type=int, default=1)
    ap.add_argument("--bucket-elems", type=int, default=1 << 27,
                    help="N > 1: bucket size of the bucketed stage-2 step (elements)")
    ap.add_argument("--c4", action="store_true",
                    help="BASELINE configs[3]: bucketed mixed ZeRO step of --optimizers "
                         "(stored-state kinds) on --model (e.g. llama-65b), one line per kind")
    ap.add_argument("--repeats", type=int, default=5,
                    help="K-step blocks per optimizer for the reported median (the first "
                         "block alone is the contract-timed value)")
    args = ap.parse_args()

    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    env_world = os.environ.get("WORLD_SIZE")
    if env_world is None and args.gpus > 1:
        sys.exit(relaunch(args.gpus))
    world = int(env_world or 1)
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per "
              "GPU (torchrun --nproc-per-node N ... --gpus N)", file=sys.stderr)
        sys.exit(2)
    rank = int(os.environ.get("RANK", 0))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    metric = "params updated/sec (all six optimizers, LLaMA-7B-shaped set)"
    config = {"workload": "configs[1]: AdamW/Lion/Adan/Sophia/LOMO+clip/AdaLomo+clip each "
                          "updating a LLaMA-7B-shaped synthetic set (291 tensors, "
                          "6,738,415,616 params)" + (
                              "; N > 1: the whole data-parallel step (gradient "
                              "reduce-scatter, update, parameter all-gather) per optimizer"
                              if world > 1 else ""),
              "model_shape": args.model, "params": None, "dtype_storage": "fp32 p/g/state",
              "grad_norm_clip": CLIP,
              "l2": "inputs larger than L2 (27 GB per buffer); no flush needed",
              "parallelism": f"dp{world} (ZeRO stage 2)" if world > 1 else "single GPU"}

    if args.impl == "reference":
        if rank != 0:
            return
        value, threads, sample, per, sec_step, n = run_cpu_reference(args.warmup, args.steps)
        config["params"] = n
        config["sample"] = sample
        line = {"impl": "reference", "metric": metric, "value": value, "unit": "params/s",
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": sec_step * 1e3, "higher_is_better": True,
                "scaling": "strong" if world > 1 else "weak",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": config,
                "cpu_baseline": {"value": value, "unit": "params/s", "cores": threads,
                                 "kind": "reference", "cpu_model": cpu_model(),
                                 "sample": sample},
                "e2e": {"value": value, "unit": "params/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0},
                "per_optimizer": per}
        print(json.dumps(line), flush=True)
        return

    import torch
    import torch.distributed as dist

    if world > 1:
        backend = os.environ.get("MCO_BENCH_BACKEND", "nccl")  # gloo: test N ranks on 1 GPU
        if backend == "nccl":
            # NCCL's init log (rank / nRanks / NVLink / NVLS lines) stays on, on stderr,
            # so the communicator actually created can be checked against --gpus
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT,NVLS")
            if torch.cuda.device_count() < world:
                print(f"bench.py: {world} ranks but {torch.cuda.device_count()} GPUs",
                      file=sys.stderr)
                sys.exit(2)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group(backend)
        local_rank = local_rank % max(torch.cuda.device_count(), 1)
    if args.c4:
        bench_c4(args, rank, world, local_rank)
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return
    res = bench_ours(args, rank, world, local_rank)
    config["params"] = res["P"]
    e2e = res.get("e2e")
    cpu = None
    if rank == 0 and world == 1 and not args.no_e2e:
        try:
            e2e = bench_e2e(args, res)
        except Exception as ex:  # report, never fake
            log(f"[e2e] failed: {ex!r}")
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            v, threads, sample, per, _, n = run_cpu_reference(1, args.cpu_steps)
            cpu = {"value": v, "unit": "params/s", "cores": threads, "kind": "reference",
                   "cpu_model": cpu_model(), "sample": sample, "params": n,
                   "per_optimizer": per}
            cpu["single_thread"] = run_cpu_single_thread()
        except Exception as ex:
            log(f"[cpu_baseline] failed: {ex!r}")
    if rank == 0:
        line = {"metric": metric, "value": res["value"], "unit": "params/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": res["ms_per_step"],
                "higher_is_better": True, "scaling": "strong" if world > 1 else "weak",
                "vs_baseline": None, "dtype": "f32", "data": "synthetic", "config": config,
                "roofline": res["roofline"], "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": res["launches"], "clocks": res["clocks"],
                "per_optimizer": res["per"]}
        if res.get("extra"):
            line["extra_not_in_value"] = res["extra"]
        if world > 1:
            line["collectives"] = {"backend": dist.get_backend(),
                                   "nccl_allgather_busbw_gbs": res["busbw"],
                                   "nvlink_nominal_gbs": NVLINK_NOMINAL_GBS}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
