#!/usr/bin/env python3
"""Optimizer-update throughput on B200: params updated / s (BASELINE.json metric).

Workload (BASELINE.json configs[1]): all six optimizers -- AdamW, Lion, Adan,
Sophia, LOMO, AdaLomo -- each updating a LLaMA-7B-shaped synthetic parameter set
(291 tensors, 6,738,415,616 fp32 params, registry order) once per step.  One
"step" = one update of the whole set by each of the six optimizers in turn;
value = 6 * P * K / (device time of the K timed steps).  Inputs are synthetic
(counter-based generator), fp32, resident in HBM, and 27 GB per buffer (> L2),
so no L2 flush is needed between iterations.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 (torchrun, one process per GPU): ZeRO partition of the same set
(ZeroPlan, parallel.cpp:20-34) -- each rank updates its owned shard; the
gradient reduce-scatter / parameter all-gather are timed separately
(`collectives`), value = P * 6 * K / max-over-ranks time ("strong").

e2e: the same metric through the C-ABI with HOST (pinned) buffers -- per step
H2D params+grads, the update, D2H params (mco_flat_step_host pipelines it for
the four stored-state kinds).  cpu_baseline / --impl reference: the
reference's own minicollie::optim (oracle/_ref, compiled from its sources)
timed on this host's cores on a bounded sample (one 7B decoder layer).
"""
from __future__ import annotations

import argparse
import gc
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

KINDS = ["adamw", "lion", "adan", "sophia", "lomo", "adalomo"]
# Algorithmic (dependency-forced) HBM bytes per parameter, fp32.
BYTES_PER_PARAM = {"adamw": 28, "lion": 20, "adan": 44, "sophia": 24, "lomo": 12,
                   "adalomo": 24}
# Paper Table 4 hyper-parameters for throughput runs; Sophia: defaults.
HPARAMS = {"adamw": dict(lr=1e-5, weight_decay=1e-2), "lion": dict(lr=3e-6, weight_decay=3e-2),
           "adan": dict(lr=5e-5, weight_decay=2e-2), "sophia": dict(lr=1e-4),
           "lomo": dict(lr=1e-2), "adalomo": dict(lr=5e-4)}


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
# reference arm / CPU baseline: the reference's own code on the host cores
# ---------------------------------------------------------------------------------------

def cpu_sample_shapes():
    from paper_2312_00407_b200.registry import CONFIG1, LLAMA_7B

    if os.environ.get("MCO_CPU_SAMPLE") == "tiny":  # CPU test of the bench contract
        return CONFIG1.shapes()[1:10]
    return LLAMA_7B.shapes()[1:10]  # one decoder layer: 9 tensors, 202,383,360 params


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def run_cpu_reference(warmup: int, steps: int):
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    from paper_2312_00407_b200.optim import OptimizerConfig, parse_kind

    if O.ref is None:
        raise RuntimeError("oracle/_ref/libmco_ref.so missing (run __graft_entry__.build())")
    shapes = cpu_sample_shapes()
    n = sum(int(__import__("math").prod(s)) for s in shapes)
    threads = host_threads()
    per = {}
    total = 0.0
    for k in KINDS:
        cfg = OptimizerConfig.defaults_for(parse_kind(k))
        for a, v in HPARAMS[k].items():
            setattr(cfg, a, v)
        sec = O.ref_bench(cfg, shapes, threads, warmup, steps)
        per[k] = {"ms": sec * 1e3, "params_per_s": n / sec}
        total += sec
        log(f"[cpu-ref] {k}: {sec * 1e3:.1f} ms/step, {n / sec / 1e9:.3f} Gparam/s "
            f"({threads} threads)")
    value = len(KINDS) * n / total
    sample = (f"one decoder layer of the registry (9 tensors, {n} fp64 params) per optimizer, "
              f"{warmup} warm-up + {steps} timed steps, one FlatOptimizer per thread over "
              "disjoint slices (stored-state kinds) / tensors across threads (LOMO, AdaLomo)")
    return value, threads, sample, per, total / max(steps, 1)


def run_cpu_single_thread():
    """The reference on ONE host thread (T = nproc and T = 1), on a
    smaller sample: the first q-projection matrix of the 7B registry."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O

    shapes = cpu_sample_shapes()[1:2]
    n = sum(int(__import__("math").prod(s)) for s in shapes)
    per, total = {}, 0.0
    for k in KINDS:
        sec = O.ref_bench(make_cfg(k), shapes, 1, 1, 1)
        per[k] = {"ms": round(sec * 1e3, 2), "params_per_s": n / sec}
        total += sec
    return {"value": len(KINDS) * n / total, "unit": "params/s", "cores": 1,
            "sample": f"one {shapes[0][0]}x{shapes[0][1]} matrix ({n} fp64 params) per "
                      "optimizer, 1 warm-up + 1 timed step", "per_optimizer": per}


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
    """One optimizer over (a shard of) the flat registry buffers, via the public API.
    N > 1: stored-state kinds and LOMO update this rank's ZeroPlan slice (gradients
    already reduced); AdaLomo runs row-split (zero.RowShardedAdaLomo) on its local
    row slices with its two statistic all-reduces inside the step."""

    def __init__(self, kind, shapes, p, g, world=1):
        import torch

        from paper_2312_00407_b200 import optim, registry, zero

        self.kind, self.p, self.g = kind, p, g
        self.cfg = make_cfg(kind)
        self.lr = self.cfg.lr
        self.rs = None
        self.n = p.numel()
        if kind in ("adamw", "lion", "adan", "sophia"):
            self.opt = optim.FlatOptimizer(self.cfg, p.numel(), device=p.device.index)
        elif kind == "adalomo" and world > 1:
            self.rs = zero.RowShardedAdaLomo(self.cfg, shapes, device=p.device.index)
            self.n = self.rs.local_numel
            self.lp = torch.empty(self.n, device=p.device)
            self.lg = torch.empty(self.n, device=p.device)
            optim.synth_fill(self.lp, registry.SEED, 0, 0xFFFE, 0, 0, -6)
            optim.synth_fill(self.lg, registry.SEED, 1, 0xFFFE, 1, 0, -7, 10)
        elif kind == "adalomo":
            self.opt = optim.AdaLomoState(self.cfg, shapes, device=p.device.index)
        else:
            self.opt = None

    def step(self):
        from paper_2312_00407_b200 import optim

        if self.kind == "lomo":
            optim.lomo_apply(self.p, self.g, self.lr, 1.0)
        elif self.rs is not None:
            self.rs.step(self.lp, self.lg, self.lr)
        elif self.kind == "adalomo":
            self.opt.apply_all(self.p, self.g, self.lr)
        else:
            self.opt.step(self.p, self.g, self.lr)


def bench_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_2312_00407_b200 import optim, registry

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    model = registry.MODELS[args.model]
    if args.layers:
        model = registry.layer_subset(model, args.layers)
    shapes = model.shapes()
    P = model.param_count()
    kinds = args.optimizers.split(",")
    hbm_peak, peak_src = measured_peaks()

    # ZeRO partition of the flat registry (N=1: the whole set)
    parts, offs = optim.zero_plan(P, world, 1)
    owned = parts[rank]
    log(f"[rank {rank}] model {model.name} P={P} owned={owned} kinds={kinds}")

    p = torch.empty(owned, dtype=torch.float32, device=dev)
    g = torch.empty(owned, dtype=torch.float32, device=dev)
    if world == 1:
        registry.fill_params(p, shapes)
        registry.fill_grads(g, shapes, 1)
    else:
        optim.synth_fill(p, registry.SEED, 0, 0xFFFF, 0, 0, -6)
        optim.synth_fill(g, registry.SEED, 1, 0xFFFF, 1, 0, -7, 10)
    torch.cuda.synchronize()

    stream = torch.cuda.current_stream()
    per = {}
    total_ms = 0.0
    launches = 0
    clocks = ClockSampler(local_rank)
    for kind in kinds:
        st = Stepper(kind, shapes, p, g, world)
        for _ in range(args.warmup):
            st.step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        l0 = optim.launch_count()
        if kind == kinds[0]:
            clocks.start()
        # per-step events (Sophia: refresh steps write h, SURVEY 8(d) reports them apart)
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
        t0 = st.opt.steps_taken() if kind in ("adamw", "lion", "adan", "sophia") else 0
        e0.record(stream)
        evs[0].record(stream)
        for i in range(args.steps):
            st.step()
            evs[i + 1].record(stream)
        e1.record(stream)
        torch.cuda.synchronize()
        launches_kind = optim.launch_count() - l0
        launches += launches_kind
        ms = e0.elapsed_time(e1) / args.steps
        step_ms = [evs[i].elapsed_time(evs[i + 1]) for i in range(args.steps)]
        # the median of repeated K-step blocks, reported next to the one
        # contract-timed block above (which alone defines ms / value)
        rep_ms = [ms]
        for _ in range(max(args.repeats, 1) - 1):
            r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            r0.record(stream)
            for _ in range(args.steps):
                st.step()
            r1.record(stream)
            torch.cuda.synchronize()
            rep_ms.append(r0.elapsed_time(r1) / args.steps)
        if world > 1:
            t = torch.tensor([ms], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = t.item()
        bpp = BYTES_PER_PARAM[kind]
        gbs = bpp * st.n / (ms * 1e-3) / 1e9  # per GPU (this rank's launch)
        per[kind] = {"ms": round(ms, 4), "params_per_s": P / (ms * 1e-3),
                     "bytes_per_param": bpp, "achieved_gbs_per_gpu": round(gbs, 1),
                     "frac_of_measured_hbm": round(gbs / hbm_peak, 4),
                     "params_per_launch": st.n,
                     "launches_per_step": args.steps and (launches_kind / args.steps),
                     "repeats": len(rep_ms), "ms_median_of_repeats":
                         round(sorted(rep_ms)[len(rep_ms) // 2], 4),
                     "ms_min_max_of_repeats": [round(min(rep_ms), 4), round(max(rep_ms), 4)]}
        if kind == "sophia":
            k = st.cfg.update_interval
            ref = [m for i, m in enumerate(step_ms) if (t0 + i) % k == 0]  # t-1 = t0+i
            non = [m for i, m in enumerate(step_ms) if (t0 + i) % k != 0]
            for name, xs, b in (("refresh", ref, 28), ("non_refresh", non, 24)):
                if xs:
                    m = sum(xs) / len(xs)
                    per[kind][name] = {"steps": len(xs), "ms": round(m, 4),
                                       "bytes_per_param": b,
                                       "frac_of_measured_hbm": round(
                                           b * st.n / (m * 1e-3) / 1e9 / hbm_peak, 4)}
        total_ms += ms
        log(f"[rank {rank}] {kind}: {ms:.3f} ms/step, {P / ms / 1e6:.1f} Gparam/s (all GPUs), "
            f"{gbs:.0f} GB/s/GPU = {gbs / hbm_peak:.3f} of {peak_src} HBM")
        del st
        gc.collect()
        torch.cuda.synchronize()
    clocks.stop()
    nk = len(per)
    value = nk * P / (total_ms * 1e-3)

    # dominant kernel = the optimizer with the largest share of the step
    dom = max(per, key=lambda k: per[k]["ms"])
    npl = per[dom]["params_per_launch"]
    kname = ("flat_tma_kernel: cp.async.bulk + mbarrier pipeline"
             if optim.flat_variant() == "tma" else f"flat_step_kernel, variant {optim.flat_variant()}")
    roofline = {"bound": "hbm", "kernel": f"{dom} update ({kname})" if dom not in (
        "lomo", "adalomo") else dom, "achieved": per[dom]["achieved_gbs_per_gpu"],
        "peak": hbm_peak, "peak_source": peak_src, "unit": "GB/s",
        "frac": round(per[dom]["achieved_gbs_per_gpu"] / hbm_peak, 4),
        "algorithmic_bytes_per_param": BYTES_PER_PARAM[dom], "params_per_launch": npl,
        "traffic": load_traffic(dom, npl)}
    out = dict(value=value, ms_per_step=total_ms, per=per, roofline=roofline,
               launches=launches, clocks=clocks.summary(), P=P, owned=owned,
               shapes=shapes, kinds=[k for k in kinds if k in per], p=p, g=g)
    out["dev"] = dev
    if world > 1 and not args.no_e2e:
        try:  # every rank takes part (max-over-ranks time); failures are reported
            out["e2e"] = bench_e2e(args, out, rank, world)
        except Exception as ex:
            log(f"[rank {rank}] e2e failed: {ex!r}")
            out["e2e"] = None
    if world > 1 and not args.no_collectives:
        del p, g
        out["p"] = out["g"] = None
        gc.collect()
        torch.cuda.empty_cache()
        try:  # the headline line must not depend on the collective benchmarks
            out["collectives"] = bench_peer_step(args, P, rank, world, dev)
        except Exception as ex:  # report, never fake
            log(f"[rank {rank}] peer-memory step unavailable: {ex!r}")
            out["collectives"] = {"unavailable": repr(ex)[:200]}
        gc.collect()
        torch.cuda.empty_cache()
        import torch.distributed as dist

        if dist.get_backend() == "nccl":  # NCCL refuses two ranks on one device (gloo tests)
            try:
                out["collectives"]["nccl_baseline"] = bench_nccl_step(args, P, rank, world, dev)
            except Exception as ex:  # report, never fake
                out["collectives"]["nccl_baseline"] = {"unavailable": repr(ex)[:200]}
    return out


def bench_nccl_step(args, P, rank, world, dev):
    """The same AdamW ZeRO step with NCCL collectives around the kernel
    (mco_shard_step: ncclReduceScatter -> owned-slice step -> ncclAllGather), the
    library-collective baseline the fused peer-memory kernel is measured against."""
    import torch
    import torch.distributed as dist

    from paper_2312_00407_b200 import optim, registry, zero

    cfg = make_cfg("adamw")
    comm = zero.NcclComm(device=dev.index)
    nz = zero.NativeZeroOptimizer(cfg, P, comm, device=dev.index)
    p = torch.empty(P, device=dev)
    g = torch.empty(P, device=dev)
    optim.synth_fill(p, registry.SEED, 0, 0xFFFC, 0, 0, -6)
    optim.synth_fill(g, registry.SEED, 1, 0xFFFC, 1, 0, -7, 10)
    for _ in range(args.warmup):
        nz.step(p, g, cfg.lr)
    torch.cuda.synchronize()
    dist.barrier()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        nz.step(p, g, cfg.lr)
    e1.record(stream)
    torch.cuda.synchronize()
    comm.check()
    ms = torch.tensor([e0.elapsed_time(e1) / args.steps], device=dev, dtype=torch.float64)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms = ms.item()
    log(f"[rank {rank}] NCCL RS + adamw + AG (mco_shard_step): {ms:.2f} ms/step")
    return {"path": "mco_shard_step: ncclReduceScatter + flat_tma_kernel + ncclAllGather",
            "ms": ms, "params_per_s": P / (ms * 1e-3)}


def bench_peer_step(args, P, rank, world, dev):
    """ZeRO step fused with its collectives (csrc/peer.cu): AdamW over the whole 7B
    set, grads summed from every rank's buffer over NVLink, params stored into every
    replica.  Roofline = max(HBM bytes / HBM BW, NVLink bytes / 770 GB/s)."""
    import torch
    import torch.distributed as dist

    from paper_2312_00407_b200 import optim, registry, zero

    cfg = make_cfg("adamw")
    ps = zero.PeerShardedOptimizer(cfg, P, device=dev.index)
    optim.synth_fill(ps.params, registry.SEED, 0, 0xFFFD, 0, 0, -6)
    optim.synth_fill(ps.grads, registry.SEED, 1, 0xFFFD, 1, 0, -7, 10)
    torch.cuda.synchronize()
    for _ in range(args.warmup):
        ps.step(cfg.lr)
    torch.cuda.synchronize()
    dist.barrier()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        ps.step(cfg.lr)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = torch.tensor([e0.elapsed_time(e1) / args.steps], device=dev, dtype=torch.float64)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms = ms.item()
    owned = ps.hi - ps.lo
    nvl = owned * (world - 1) * 4 / 1e9  # GB in (grads) and out (params) per rank
    hbm = owned * (28 + 4 * world) / 1e9  # local state + master + grads + replica traffic
    bound_ms = max(nvl / 770.0, hbm / measured_peaks()[0]) * 1e3
    log(f"[rank {rank}] fused RS+adamw+AG: {ms:.2f} ms/step, NVLink {nvl:.1f} GB/dir/rank, "
        f"roofline {bound_ms:.2f} ms")
    return {"kernel": "peer_step_kernel (adamw, RS + update + AG over NVLink)", "ms": ms,
            "params_per_s": P / (ms * 1e-3), "nvlink_gb_per_direction_per_rank": round(nvl, 2),
            "roofline_ms": round(bound_ms, 3), "frac": round(bound_ms / ms, 4),
            "nvlink_peak_gbs": 770.0}


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
    """Host-buffer end-to-end: per step H2D(p, g) + update + D2H(p).  N > 1: every rank
    runs its own part (the ZeroPlan slice for the flat kinds and LOMO, every N-th tensor
    for AdaLomo) through the same host-span calls over its own PCIe link; per-kind time =
    max over ranks; bytes are whole-job."""
    import math

    import psutil
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
    n_ada = sum(int(math.prod(s)) for s in shapes)
    need = 2 * max(P, n_ada) * 4 * 1.3
    avail = psutil.virtual_memory().available / world
    fits = need < avail * 0.6
    n = P
    if world == 1 and not fits:  # whole tensors prefix that fits
        cap = int(avail * 0.6 / (2 * 4 * 1.3)) // 1024 * 1024
        acc, k = 0, 0
        while k < len(shapes) and acc + int(math.prod(shapes[k])) <= cap:
            acc += int(math.prod(shapes[k]))
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
    src_p, src_g = res["p"][:n].cpu(), res["g"][:n].cpu()
    for a in range(0, m, n):  # the part's values, repeated when AdaLomo's subset is larger
        b = min(m, a + n)
        hp[a:b].copy_(src_p[:b - a])
        hg[a:b].copy_(src_g[:b - a])
    del src_p, src_g
    pcie = pcie_ceiling(hp, res["p"].device)
    log(f"[e2e] rank {rank}: PCIe ceiling (pinned, GB/s): {pcie}")
    steps = max(1, min(args.steps, args.e2e_steps))
    tot_s, h2d, d2h, h2d_me, d2h_me = 0.0, 0, 0, 0, 0
    per = {}
    opt = ada = one = None
    for kind in res["kinds"]:
        cfg = make_cfg(kind)
        opt = ada = one = None  # free the previous optimizer's device state first
        gc.collect()
        k_n = n_ada if kind == "adalomo" else n
        hpn, hgn = hp[:k_n].numpy(), hg[:k_n].numpy()
        if kind in ("adamw", "lion", "adan", "sophia"):
            opt = optim.FlatOptimizer(cfg, k_n)

            def one():
                opt.step(hpn, hgn, cfg.lr)  # mco_flat_step_host: pipelined H2D/step/D2H
        elif kind == "adalomo":
            ada = optim.AdaLomoState(cfg, shapes)

            def one():
                ada.apply_all(hpn, hgn, cfg.lr)  # per-tensor H2D / apply / D2H pipeline
        else:
            def one():
                optim.lomo_apply(hpn, hgn, cfg.lr, 1.0)  # mco_lomo_apply_host
        one()
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        for _ in range(steps):
            one()
        torch.cuda.synchronize()
        dt = max_over_ranks((time.perf_counter() - t0) / steps)
        total = res["P"] if world > 1 else k_n  # params of the whole job this step
        per[kind] = {"ms": round(dt * 1e3, 2), "params_per_s": total / dt}
        tot_s += dt
        h2d += 2 * total * 4
        d2h += total * 4
        h2d_me += 2 * k_n * 4
        d2h_me += k_n * 4
        if rank == 0:
            log(f"[e2e] {kind}: {dt * 1e3:.1f} ms/step, {total / dt / 1e9:.2f} Gparam/s")
    # the copies bound the step: max(H2D bytes / H2D BW, D2H / D2H BW, all / both-ways BW)
    # over this rank's own link (every rank has one)
    bound_s = max(h2d_me / (pcie["h2d_gbs"] * 1e9), d2h_me / (pcie["d2h_gbs"] * 1e9),
                  (h2d_me + d2h_me) / (pcie["both_gbs"] * 1e9))
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
                    "mco_lomo_apply_host, mco_adalomo_apply_all_host (H2D p+g, update, D2H p "
                    "pipelined per chunk / per tensor)" + (
                        f"; each of {world} ranks over its own part" if world > 1 else "")}


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
    ap.add_argument("--no-collectives", action="store_true")
    ap.add_argument("--cpu-steps", type=int, default=2)
    ap.add_argument("--repeats", type=int, default=5,
                    help="K-step blocks per optimizer for the reported median (the first "
                         "block alone is the contract-timed value)")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    metric = "params updated/sec (all six optimizers, LLaMA-7B-shaped set)"
    config = {"workload": "configs[1]: AdamW/Lion/Adan/Sophia/LOMO/AdaLomo each updating a "
                          "LLaMA-7B-shaped synthetic set (291 tensors, 6,738,415,616 params)",
              "model_shape": args.model, "params": None, "dtype_storage": "fp32 p/g/state",
              "l2": "inputs larger than L2 (27 GB per buffer); no flush needed",
              "parallelism": f"zero{world}" if world > 1 else "single GPU"}

    if args.impl == "reference":
        if rank != 0:
            return
        value, threads, sample, per, sec_step = run_cpu_reference(args.warmup, args.steps)
        from paper_2312_00407_b200.registry import LLAMA_7B

        config["params"] = LLAMA_7B.param_count()
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
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group(backend)
        local_rank = local_rank % max(torch.cuda.device_count(), 1)
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
            v, threads, sample, per, _ = run_cpu_reference(1, args.cpu_steps)
            cpu = {"value": v, "unit": "params/s", "cores": threads, "kind": "reference",
                   "cpu_model": cpu_model(), "sample": sample, "per_optimizer": per}
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
        if "collectives" in res:
            line["collectives"] = res["collectives"]
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
