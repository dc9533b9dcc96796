"""ZeRO sharding of the optimizer step across GPUs (one process per GPU).

Reference: the optimizer section of ParallelWorker (parallel.cpp:326-339 creation,
626-681 step) over ZeroPlan (parallel.cpp:20-38).  North-star flow
("ZeRO-1 style ... RS grads, AG params") = the reference's stage-2 branch
(parallel.cpp:656-666):

    owned_grads = reduce_scatter(flat_grads, SUM, plan.part_sizes)   # :657-658
    FlatOptimizer::step(params[owned], owned_grads, lr)                # :660
    params = all_gather(params[owned])                                 # :661-663

Partition bookkeeping is ZeroPlan's, bit for bit (first P % N ranks own one
more element).  Collectives go through torch.distributed: NCCL over NVLink on
B200, gloo in the CPU tests.  Equal parts use reduce_scatter_tensor /
all_gather_into_tensor; unequal parts (P % N != 0) fall back to one
reduce / broadcast per part, which keeps the reference's ownership exactly.
The grad reduction is a SUM, as the reference's (the backward seed already
carries 1/global_count, parallel.cpp:516-522, 602).

The single-kernel alternative -- reduce-scatter, update and all-gather fused
over NVLink peer memory -- is `PeerShardedOptimizer` (csrc/peer.cu).
"""
from __future__ import annotations

from typing import Callable, Optional

from . import optim


def _dist():
    import torch.distributed as dist

    return dist


def check_agreement(what: str, fields: dict, group=None) -> None:
    """Every rank must build its sharded optimizer from the same plan (total length,
    kind, shapes ...).  One all_gather_object at construction; on a mismatch EVERY
    rank raises ProtocolError naming the disagreeing ranks -- instead of hanging in
    (or silently mis-pairing) the per-step collectives.  The reference aborts a
    collective whose members disagree on the length (comm.cpp:160-167) and re-raises
    worker failures with a [rank r] prefix (comm.cpp:337-360)."""
    dist = _dist()
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return
    world = dist.get_world_size(group)
    mine = tuple(sorted((k, repr(v)) for k, v in fields.items()))
    allf = [None] * world
    dist.all_gather_object(allf, mine, group=group)
    bad = [r for r in range(world) if allf[r] != allf[0]]
    if bad:
        diff = {r: dict(allf[r]) for r in [0] + bad}
        raise optim.ProtocolError(
            f"[rank {dist.get_rank(group)}] {what}: ranks {bad} disagree with rank 0: {diff}")


class ZeroPlan:
    """parallel.hpp:22-29 / parallel.cpp:20-38 (computed by the C-ABI, mco_zero_plan)."""

    def __init__(self, total_len: int, dp_size: int, stage: int = 2):
        self.stage = stage
        self.part_sizes, self.offsets = optim.zero_plan(total_len, dp_size, stage)

    @staticmethod
    def make(total_len: int, dp_size: int, stage: int = 2) -> "ZeroPlan":
        return ZeroPlan(total_len, dp_size, stage)

    def owned_range(self, dp_index: int) -> tuple[int, int]:
        return self.offsets[dp_index], self.offsets[dp_index + 1]

    @property
    def even(self) -> bool:
        return len(set(self.part_sizes)) <= 1


def phased_empty(n: int, dtype, device, phase: int):
    """An n-element buffer whose first element sits `phase` elements past a 32 B
    boundary (mod 8 elements): gradients reduced for a shard view at an odd offset share
    its alignment phase, so the update kernel peels a short head and vectorises the rest
    (flat.cu launch_flat_step) instead of running every element on the scalar path."""
    import torch

    buf = torch.empty(n + 8, dtype=dtype, device=device)
    shift = (phase - (buf.data_ptr() // buf.element_size())) % 8
    return buf[shift:shift + n]


def elem_phase(t) -> int:
    return (t.data_ptr() // t.element_size()) % 8


def _gloo_cuda(t, group) -> bool:
    return t.is_cuda and _dist().get_backend(group) == "gloo"


def rs_tensor(out, inp, group=None) -> None:
    """reduce_scatter_tensor(SUM).  gloo has no CUDA reduce-scatter (it is the backend of
    the several-ranks-on-one-GPU tests): all-reduce a copy and keep this rank's chunk."""
    dist = _dist()
    if _gloo_cuda(inp, group):
        tmp = inp.clone()
        dist.all_reduce(tmp, op=dist.ReduceOp.SUM, group=group)
        r, n = dist.get_rank(group), out.numel()
        out.copy_(tmp[r * n:(r + 1) * n])
        return
    dist.reduce_scatter_tensor(out, inp, op=dist.ReduceOp.SUM, group=group)


def ag_tensor(out, inp, group=None) -> None:
    """all_gather_into_tensor; gloo + CUDA: an all-reduce of zeros around this rank's
    chunk (x + 0 == x exactly)."""
    dist = _dist()
    if _gloo_cuda(inp, group):
        import torch

        r, n = dist.get_rank(group), inp.numel()
        tmp = torch.zeros_like(out)
        tmp[r * n:(r + 1) * n].copy_(inp)
        dist.all_reduce(tmp, op=dist.ReduceOp.SUM, group=group)
        out.copy_(tmp)
        return
    dist.all_gather_into_tensor(out, inp, group=group)


def reduce_scatter_owned(flat, plan: ZeroPlan, rank: int, group=None, phase: int = 0):
    """SUM-reduce `flat` and return this rank's owned slice (comm.cpp:219-246 semantics),
    in a buffer of the given alignment phase."""
    dist = _dist()
    lo, hi = plan.owned_range(rank)
    world = len(plan.part_sizes)
    if world == 1:
        return flat[lo:hi]
    if plan.even:
        out = phased_empty(hi - lo, flat.dtype, flat.device, phase)
        rs_tensor(out, flat, group)
        return out
    out = None
    for r in range(world):
        a, b = plan.owned_range(r)
        part = phased_empty(b - a, flat.dtype, flat.device, phase if r == rank else 0)
        part.copy_(flat[a:b])
        if _gloo_cuda(part, group):
            dist.all_reduce(part, op=dist.ReduceOp.SUM, group=group)
        else:
            dist.reduce(part, dst=dist.get_global_rank(group, r) if group else r,
                        op=dist.ReduceOp.SUM, group=group)
        if r == rank:
            out = part
    return out


def all_gather_owned(flat, plan: ZeroPlan, rank: int, group=None) -> None:
    """In place: every rank's owned slice of `flat` broadcast to all (comm.cpp:207-217)."""
    dist = _dist()
    world = len(plan.part_sizes)
    if world == 1:
        return
    lo, hi = plan.owned_range(rank)
    if plan.even:
        ag_tensor(flat[:plan.offsets[-1]], flat[lo:hi].clone(), group)
        return
    for r in range(world):
        a, b = plan.owned_range(r)
        view = flat[a:b]
        buf = view.clone() if not view.is_contiguous() else view
        dist.broadcast(buf, src=dist.get_global_rank(group, r) if group else r, group=group)


class ZeroShardedOptimizer:
    """Sharded stored-state optimizer (AdamW / Lion / Adan / Sophia).

    Each rank keeps optimizer state (and, with `mixed`, an fp32 master copy) for
    its ZeroPlan-owned slice only.  flat_params are replicated (fp32, or bf16 when
    mixed); flat_grads are each rank's local (unreduced) gradients.

    local_step(p_owned, g_owned, lr, p_out_owned) defaults to the CUDA
    FlatOptimizer over the owned slice; tests on CPU inject the oracle.
    """

    def __init__(self, cfg: optim.OptimizerConfig, total_len: int, group=None, stage: int = 2,
                 mixed: bool = False, master_init=None, device: Optional[int] = None,
                 local_step: Optional[Callable] = None):
        dist = _dist()
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        check_agreement("ZeroShardedOptimizer", dict(total_len=total_len, stage=stage,
                                                     kind=int(cfg.kind), mixed=mixed), group)
        self.plan = ZeroPlan.make(total_len, self.world, stage)
        self.stage = stage
        self.total_len = total_len
        # the optimizer owns the ZeroPlan part for stage >= 1, everything at stage 0
        # (parallel.cpp:330)
        self.lo, self.hi = self.plan.owned_range(self.rank) if stage >= 1 else (0, total_len)
        self.mixed = mixed
        self.master = None
        if mixed:
            if master_init is None:
                raise optim.ContractError("mixed sharding needs the fp32 master init slice")
            self.master = master_init[self.lo:self.hi].float().clone()
        self._local = local_step
        if local_step is None:
            dev = optim._device(device)
            self.opt = optim.FlatOptimizer(cfg, self.hi - self.lo, device=dev)
        else:
            self.opt = None

    def step(self, flat_params, flat_grads, lr: float) -> None:
        """The ZeRO branches of ParallelWorker::train_step (parallel.cpp:637-672):
          stage 0: all-reduce(SUM) grads, step the whole vector on every rank;
          stage 1: all-reduce(SUM) grads, step the owned slice, all-gather params;
          stage 2: reduce-scatter(SUM) grads, step the owned slice, all-gather params;
          stage 3: reduce-scatter(SUM) grads, step the owned shard -- flat_params IS
                   this rank's shard (hi - lo elements), nothing is gathered.
        Stages 0 and 1 reduce flat_grads in place (as the reference reduces its
        flattened copy); stages 2 and 3 leave it untouched."""
        if self.stage == 3:
            if flat_params.numel() != self.hi - self.lo:
                raise optim.ContractError(
                    f"zero stage 3: params hold {flat_params.numel()} elements, the owned "
                    f"shard is {self.hi - self.lo}")
        elif flat_params.numel() != self.total_len or flat_grads.numel() != self.total_len:
            raise optim.ContractError(
                f"zero step: flat buffers of {flat_params.numel()} / {flat_grads.numel()} "
                f"elements for a plan of {self.total_len}")
        if self.stage <= 1:
            if self.world > 1:
                dist = _dist()
                dist.all_reduce(flat_grads, op=dist.ReduceOp.SUM, group=self.group)
            g_owned = flat_grads[self.lo:self.hi]
        p_owned = flat_params if self.stage == 3 else flat_params[self.lo:self.hi]
        if (self.mixed and self.master.is_cuda and self._local is None
                and elem_phase(self.master) != elem_phase(p_owned)):
            # the fp32 master moves to the bf16 replica slice's alignment phase (once,
            # before the state takes the master's phase at the first step)
            m = phased_empty(self.master.numel(), self.master.dtype, self.master.device,
                             elem_phase(p_owned))
            m.copy_(self.master)
            self.master = m
        if self.stage >= 2:
            ref = self.master if self.mixed else p_owned
            g_owned = reduce_scatter_owned(flat_grads, self.plan, self.rank, self.group,
                                           phase=elem_phase(ref) if ref.is_cuda else 0)
        if self._local is not None:
            self._local(self.master if self.mixed else p_owned, g_owned, lr,
                        p_owned if self.mixed else None)
        elif self.mixed:
            self.opt.step_mixed(self.master, g_owned.contiguous(), p_owned, lr)
        else:
            self.opt.step(p_owned, g_owned.contiguous(), lr)
        if self.stage in (1, 2):
            all_gather_owned(flat_params, self.plan, self.rank, self.group)

    def owned_range(self) -> tuple[int, int]:
        return self.lo, self.hi

    # checkpoint hand-off by buffer name (parallel.cpp:820-862)
    def extract_state(self) -> dict:
        out = {"steps": self.opt.steps_taken() if self.opt else 0, "buffers": {}}
        if self.opt is not None:
            for name, t in self.opt.buffers():
                out["buffers"][name] = t.clone()
        return out

    def load_state(self, state: dict) -> None:
        if self.opt is None:
            return
        for name, t in self.opt.buffers():
            src = state["buffers"].get(name)
            if src is not None and src.numel() == t.numel():  # match by name and size
                t.copy_(src)
        self.opt.set_steps_taken(state["steps"])


class _CudaLomoOps:
    sumsq = staticmethod(optim.sumsq)
    apply = staticmethod(optim.lomo_apply)
    apply_clipped = staticmethod(optim.lomo_apply_clipped)


def sharded_lomo_step(p_owned, g_owned, lr: float, clip: Optional[float], group=None,
                      stream=None, ops=_CudaLomoOps):
    """LOMO over ZeRO shards with the global grad-norm clip (C5): local sum of
    squares -> all_reduce(SUM) of one fp64 scalar -> scaled update.  The
    reference forbids clipping in parallel runs (parallel.cpp:335-337); this is
    the serial rule (optim.cpp:291-303) on the concatenated gradient.
    `ops` is the kernel set (CUDA by default; CPU tests inject the oracle)."""
    dist = _dist()
    if clip is None:
        ops.apply(p_owned, g_owned, lr, 1.0, stream)
        return None
    s = ops.sumsq(g_owned, stream=stream)
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(s, op=dist.ReduceOp.SUM, group=group)
    ops.apply_clipped(p_owned, g_owned, lr, s, clip, stream)
    return s


class _PeerBuffer:
    """A cudaMalloc'ed flat buffer whose CUDA IPC handle can be shared."""

    def __init__(self, numel: int, dtype, device: int):
        import ctypes as C

        from ._lib import lib

        self.numel, self.dtype, self.device = numel, dtype, device
        self.esize = {"float32": 4, "bfloat16": 2}[str(dtype).split(".")[-1]]
        self._free = lib.mco_peer_free  # kept: module globals vanish at shutdown
        p = C.c_void_p()
        optim._check(lib.mco_peer_alloc(numel * self.esize, device, C.byref(p)))
        self.ptr = p.value

    def tensor(self):
        import torch

        code = optim.MCO_F32 if self.esize == 4 else optim.MCO_BF16
        if code == optim.MCO_F32:
            return optim._as_tensor(self.ptr, self.numel, optim.MCO_F32, self, self.device)
        raw = torch.as_tensor(_U16View(self.ptr, self.numel, self), device=f"cuda:{self.device}")
        return raw.view(torch.bfloat16)

    def handle(self) -> bytes:
        import ctypes as C

        from ._lib import lib

        buf = (C.c_char * 64)()
        optim._check(lib.mco_peer_export(self.ptr, buf))
        return bytes(buf)

    def __del__(self):
        if getattr(self, "ptr", None):
            self._free(self.ptr)
            self.ptr = None


class _U16View:
    def __init__(self, ptr, n, owner):
        self._owner = owner
        self.__cuda_array_interface__ = {"shape": (int(n),), "typestr": "<i2",
                                         "data": (int(ptr), False), "version": 3,
                                         "strides": None, "stream": None}


class PeerBuffers:
    """This rank's symmetric flat parameter replica + gradient buffer, and every
    rank's mapping of them (CUDA IPC handles exchanged over the process group).
    On one device with several processes (tests) the same IPC path is used."""

    def __init__(self, total_len: int, group=None, param_dtype=None, grad_dtype=None,
                 device: Optional[int] = None):
        import ctypes as C

        import torch

        from ._lib import lib

        dist = _dist()
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.device = device = optim._device(device)
        self.total_len = total_len
        check_agreement("PeerBuffers", dict(total_len=total_len, param_dtype=str(param_dtype),
                                            grad_dtype=str(grad_dtype)), group)
        self._pbuf = _PeerBuffer(total_len, param_dtype or torch.float32, device)
        self._gbuf = _PeerBuffer(total_len, grad_dtype or torch.float32, device)
        self.params, self.grads = self._pbuf.tensor(), self._gbuf.tensor()
        mine = (self._pbuf.handle(), self._gbuf.handle())
        if self.world > 1:
            allh = [None] * self.world
            dist.all_gather_object(allh, mine, group=group)
        else:
            allh = [mine]
        self._opened = []
        self._close = lib.mco_peer_close
        self.pptrs, self.gptrs = [], []
        for r, (ph, gh) in enumerate(allh):
            if r == self.rank:
                self.pptrs.append(self._pbuf.ptr)
                self.gptrs.append(self._gbuf.ptr)
                continue
            pp, gp = C.c_void_p(), C.c_void_p()
            optim._check(lib.mco_peer_import(C.c_char_p(ph), device, C.byref(pp)))
            optim._check(lib.mco_peer_import(C.c_char_p(gh), device, C.byref(gp)))
            self._opened += [pp.value, gp.value]
            self.pptrs.append(pp.value)
            self.gptrs.append(gp.value)
        self.pdt = optim._dtype_code(self.params)
        self.gdt = optim._dtype_code(self.grads)

    def barrier(self) -> None:
        """Order the ranks around a peer kernel.  NCCL: a one-element all-reduce on
        the stream (no host sync).  Other backends: host sync + barrier."""
        import torch

        dist = _dist()
        if self.world == 1:
            return
        if dist.get_backend(self.group) == "nccl":
            dist.all_reduce(torch.zeros(1, device=self.params.device), group=self.group)
        else:
            torch.cuda.synchronize()
            dist.barrier(group=self.group)

    def __del__(self):
        close = getattr(self, "_close", None)
        for p in getattr(self, "_opened", []):
            close(p)


class PeerShardedOptimizer:
    """ZeRO step as ONE kernel per rank over NVLink peer memory (csrc/peer.cu):
    the owned slice's gradients are summed straight out of every rank's grad
    buffer, the update runs, and the new parameters are stored straight into
    every rank's replica -- no reduced-gradient buffer, no separate NCCL
    reduce-scatter / all-gather.  Same ZeroPlan ownership and same result as
    ZeroShardedOptimizer (SUM of grads in rank order).

    Write gradients into `self.grads`, call step(lr), read `self.params`.
    Stored-state kinds keep state (+ fp32 master for bf16 replicas) for the owned
    slice; LOMO keeps nothing (optionally the global-norm clip, C5).
    """

    def __init__(self, cfg: optim.OptimizerConfig, total_len: int, group=None,
                 param_dtype=None, grad_dtype=None, master_init=None, device: Optional[int] = None,
                 buffers: Optional[PeerBuffers] = None):
        self.cfg = cfg
        self.buf = buffers or PeerBuffers(total_len, group, param_dtype, grad_dtype, device)
        b = self.buf
        self.world, self.rank = b.world, b.rank
        self.params, self.grads = b.params, b.grads
        self.plan = ZeroPlan.make(total_len, self.world, 2)
        self.lo, self.hi = self.plan.owned_range(self.rank)
        if b.pdt == optim.MCO_F32 and master_init is None:
            self.master = self.params[self.lo:self.hi]  # the f32 replica is the master
        else:
            src = master_init if master_init is not None else self.params
            self.master = src[self.lo:self.hi].float().contiguous().clone()
        self.lomo = cfg.kind == optim.Kind.LOMO
        self.opt = None if self.lomo else optim.FlatOptimizer(cfg, self.hi - self.lo,
                                                              device=device)
        self._norm = None

    def step(self, lr: float, stream=None) -> None:
        import ctypes as C

        import torch

        from ._lib import lib

        b = self.buf
        b.barrier()  # every rank's gradients are final
        if self.lomo:
            n = self.hi - self.lo
            ga = (C.c_void_p * self.world)(*b.gptrs)
            pa = (C.c_void_p * self.world)(*b.pptrs)
            sumsq = None
            if self.cfg.clip_threshold is not None:
                if self._norm is None:
                    self._norm = torch.zeros((), dtype=torch.float64, device=self.params.device)
                optim._check(lib.mco_sumsq_peers(ga, b.gdt, self.world, self.lo, n,
                                                 self._norm.data_ptr(), optim._stream(stream)))
                if self.world > 1:
                    _dist().all_reduce(self._norm, group=b.group)
                sumsq = self._norm.data_ptr()
            optim._check(lib.mco_lomo_apply_peers(
                ga, b.gdt, pa, b.pdt, self.world, self.master.data_ptr(), self.lo, n, float(lr),
                1.0, sumsq, float(self.cfg.clip_threshold or 0.0), optim._stream(stream)))
        else:
            self.opt.step_peers(b.gptrs, b.pptrs, self.master, self.lo, self.hi - self.lo, lr,
                                grad_dtype=b.gdt, param_dtype=b.pdt, stream=stream)
        b.barrier()  # every replica is complete


class RowShardedAdaLomo:
    """AdaLomo with every matrix split by rows across the ranks (SURVEY 8(e), C3 at
    8 GPUs); 1-D tensors are replicated.  Row slices follow ZeroPlan over each
    matrix's rows.  Per step, two all-reduces (SUM) of fp64 payloads:
      1. per-tensor [sum g^2, sum p^2, sum v_row_old] + every matrix's column sums
         (the column statistics of a row-split matrix, optim.cpp:241-249),
      2. per-tensor sum u^2 (the update-RMS damping, optim.cpp:269-272).
    Row statistics stay local (rows are whole on a rank).  Replicated tensors
    contribute from rank 0 only (weight 0 elsewhere) and are updated identically
    everywhere.  The reference's own TP variant computes stats per local shard
    (parallel.cpp:334, 593-594) and is NOT serial AdaLomo; this is."""

    def __init__(self, cfg: optim.OptimizerConfig, shapes, group=None, device: Optional[int] = None,
                 rank: Optional[int] = None, world: Optional[int] = None,
                 grad_clip: Optional[float] = None):
        """grad_clip: the global grad-norm clip over the whole (all-rank) gradient
        (C3; the LOMO rule, optim.cpp:302-303, on the concatenated gradient): the
        per-rank Σg² rides in the first all-reduce payload."""
        dist = _dist()
        self.group = group
        if world is None:  # explicit rank/world: single-process (virtual-rank) use
            world = dist.get_world_size(group) if dist.is_initialized() else 1
            rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world, self.rank = world, rank
        self.global_shapes = [tuple(s) for s in shapes]
        if dist.is_initialized() and self.world > 1:
            check_agreement("RowShardedAdaLomo", dict(shapes=self.global_shapes,
                                                      kind=int(cfg.kind), grad_clip=grad_clip),
                            group)
        self.local_shapes, self.pieces, self._shard = [], [], []
        goff = 0
        for s in self.global_shapes:
            n = 1
            for d in s:
                n *= d
            if len(s) == 2:
                parts, offs = optim.zero_plan(s[0], self.world, 1)
                r0, r1 = offs[self.rank], offs[self.rank + 1]
                self.local_shapes.append((r1 - r0, s[1]))
                self.pieces.append((goff + r0 * s[1], (r1 - r0) * s[1]))
                self._shard.append((s[0], 1.0))
            else:
                self.local_shapes.append(s)
                self.pieces.append((goff, n))
                self._shard.append((s[0] if s else 1, 1.0 if self.rank == 0 else 0.0))
            goff += n
        self.state = optim.AdaLomoState(cfg, self.local_shapes, device=device,
                                        grad_clip=grad_clip)
        for k, (rows, w) in enumerate(self._shard):
            self.state.set_shard(k, rows, w)
        self.local_numel = int(self.state.offsets[-1])

    def scatter(self, flat_global):
        """This rank's local flat buffer (registry order of local slices)."""
        import torch

        return torch.cat([flat_global[a:a + n] for a, n in self.pieces])

    def gather_into(self, local, flat_global) -> None:
        off = 0
        for a, n in self.pieces:
            flat_global[a:a + n].copy_(local[off:off + n])
            off += n

    def step(self, local_p, local_g, lr: float, stream=None) -> None:
        dist = _dist()
        multi = self.world > 1 and dist.is_initialized()
        self.state.phase(1, local_p, local_g, lr, stream)
        if multi:
            dist.all_reduce(self.state.payload(0), op=dist.ReduceOp.SUM, group=self.group)
        self.state.phase(2, local_p, local_g, lr, stream)
        if multi:
            dist.all_reduce(self.state.payload(1), op=dist.ReduceOp.SUM, group=self.group)
        self.state.phase(3, local_p, local_g, lr, stream)

    # ---- data-parallel form: gradients reduced and parameters gathered in the step ----
    # Rank-major layout: chunk q (q = 0..world-1, `chunk` elements each, zero padded)
    # holds rank q's local buffer (its row slices + every replicated 1-D tensor, in
    # registry order).  A reduce-scatter(SUM) of each rank's local gradients in this
    # layout hands rank r exactly the summed gradient of its rows and of the replicated
    # tensors; an all-gather of the chunks rebuilds every rank's replica.

    @staticmethod
    def local_len_of(shapes, world: int, rank: int) -> int:
        n = 0
        for s in shapes:
            if len(s) == 2:
                _, offs = optim.zero_plan(s[0], world, 1)
                n += (offs[rank + 1] - offs[rank]) * s[1]
            else:
                k = 1
                for d in s:
                    k *= d
                n += k
        return n

    @staticmethod
    def chunk_len(shapes, world: int) -> int:
        """Rank-major chunk length: the largest rank's local buffer."""
        return max(RowShardedAdaLomo.local_len_of(shapes, world, r) for r in range(world))

    def local_len(self, rank: int) -> int:
        return self.local_len_of(self.global_shapes, self.world, rank)

    @property
    def chunk(self) -> int:
        if not hasattr(self, "_chunk"):
            self._chunk = self.chunk_len(self.global_shapes, self.world)
        return self._chunk

    def pieces_of(self, rank: int):
        """(global offset, length) of rank's local pieces, registry order."""
        out, goff = [], 0
        for s in self.global_shapes:
            n = 1
            for d in s:
                n *= d
            if len(s) == 2:
                _, offs = optim.zero_plan(s[0], self.world, 1)
                out.append((goff + offs[rank] * s[1], (offs[rank + 1] - offs[rank]) * s[1]))
            else:
                out.append((goff, n))
            goff += n
        return out

    def to_rank_major(self, flat_global, out=None):
        """Registry-order flat buffer -> rank-major (world x chunk)."""
        import torch

        c = self.chunk
        if out is None:
            out = torch.zeros(self.world * c, dtype=flat_global.dtype, device=flat_global.device)
        for r in range(self.world):
            off = r * c
            for a, n in self.pieces_of(r):
                out[off:off + n].copy_(flat_global[a:a + n])
                off += n
        return out

    def from_rank_major(self, rm, flat_global) -> None:
        """Rank-major -> registry order (replicated tensors taken from chunk 0)."""
        c = self.chunk
        for r in range(self.world):
            off = r * c
            for a, n in self.pieces_of(r):
                flat_global[a:a + n].copy_(rm[off:off + n])
                off += n

    def step_dp(self, rm_params, rm_grads, lr: float, stream=None) -> None:
        """One data-parallel AdaLomo step (C3 at N GPUs): reduce-scatter(SUM) of the
        rank-major local gradients -> phase 1 -> all-reduce statistics payload (column
        sums, Σg² for the clip, Σp², Σv_row) -> phase 2 -> all-reduce Σu² payload ->
        phase 3 on this rank's rows -> all-gather of the rank-major parameters.  Equals
        serial AdaLomo (optim.cpp:215-275, clip: optim.cpp:302-303) on the summed
        gradient; the reference's TP variant (parallel.cpp:334, 593-594) does not."""
        dist = _dist()
        c, n = self.chunk, self.local_numel
        if rm_params.numel() != self.world * c or rm_grads.numel() != self.world * c:
            raise optim.ContractError(
                f"row-sharded adalomo: rank-major buffers of {rm_params.numel()} / "
                f"{rm_grads.numel()} elements, expected {self.world} x {c}")
        lo = self.rank * c
        local_p = rm_params[lo:lo + n]
        if self.world > 1 and dist.is_initialized():
            if not hasattr(self, "_gred") or self._gred.dtype != rm_grads.dtype:
                self._gred = phased_empty(c, rm_grads.dtype, rm_grads.device,
                                          elem_phase(local_p))
            rs_tensor(self._gred, rm_grads, self.group)
            local_g = self._gred[:n]
        else:
            local_g = rm_grads[lo:lo + n]
        self.step(local_p, local_g, lr, stream)
        if self.world > 1 and dist.is_initialized():
            ag_tensor(rm_params, rm_params[lo:lo + c].clone(), self.group)


class ZeroShardedLomo:
    """LOMO (optionally with the global grad-norm clip, C5) as a data-parallel ZeRO
    step: reduce-scatter(SUM) of the flat gradients over ZeroPlan parts -> local Σg² ->
    all-reduce of one fp64 scalar -> clipped update of the owned slice -> all-gather of
    the parameters (parallel.cpp:656-666 with LOMO in place of FlatOptimizer; the
    reference forbids the clip in parallel runs, parallel.cpp:335-337, this applies the
    serial rule, optim.cpp:291-303, to the summed gradient)."""

    def __init__(self, total_len: int, clip: Optional[float] = None, group=None,
                 ops=_CudaLomoOps):
        dist = _dist()
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        check_agreement("ZeroShardedLomo", dict(total_len=total_len, clip=clip), group)
        self.plan = ZeroPlan.make(total_len, self.world, 2)
        self.lo, self.hi = self.plan.owned_range(self.rank)
        self.total_len, self.clip, self.ops = total_len, clip, ops

    def step(self, flat_params, flat_grads, lr: float, stream=None):
        if flat_params.numel() != self.total_len or flat_grads.numel() != self.total_len:
            raise optim.ContractError(
                f"zero lomo step: flat buffers of {flat_params.numel()} / "
                f"{flat_grads.numel()} elements for a plan of {self.total_len}")
        p_owned = flat_params[self.lo:self.hi]
        g_owned = reduce_scatter_owned(flat_grads, self.plan, self.rank, self.group,
                                       phase=elem_phase(p_owned) if p_owned.is_cuda else 0)
        s = sharded_lomo_step(p_owned, g_owned, lr, self.clip, self.group, stream, self.ops)
        all_gather_owned(flat_params, self.plan, self.rank, self.group)
        return s


def reshard_state(states: list, total_len: int, new_world: int) -> list:
    """Offline reshard of ZeRO optimizer state (the reference's gather_full_params +
    load_state contract, parallel.cpp:820-935): `states[r]` is rank r's
    extract_state() under ZeroPlan(total_len, len(states)); returns the
    extract_state()-shaped dicts for ZeroPlan(total_len, new_world).  Buffers are
    matched by name (m, v, n, h, g_prev); the step counter must agree."""
    import torch

    steps = {s["steps"] for s in states}
    if len(steps) != 1:
        raise optim.ContractError("reshard: ranks disagree on the step counter")
    names = list(states[0]["buffers"])
    full = {}
    for name in names:
        parts = [s["buffers"][name] for s in states]
        full[name] = torch.cat([p.reshape(-1) for p in parts])
        if full[name].numel() != total_len:
            raise optim.ContractError(f"reshard: buffer '{name}' does not cover the set")
    plan = ZeroPlan.make(total_len, new_world)
    out = []
    for r in range(new_world):
        lo, hi = plan.owned_range(r)
        out.append({"steps": states[0]["steps"],
                    "buffers": {n: full[n][lo:hi].clone() for n in names}})
    return out


class NcclComm:
    """The C-ABI's own NCCL communicator (mco_comm): ncclUniqueId from rank 0, shipped
    over the torch.distributed group (any backend), ncclCommInitRank on every rank.
    Lets the sharded step run as one stream-ordered C call (mco_shard_step).

    timeout_s: the communicator's deadline (mco_comm_create_timeout; None = the
    library default, $MCO_NCCL_TIMEOUT_S or 600 s).  world / rank / unique_id: build it
    without a process group (the id must then be shared by the caller)."""

    def __init__(self, group=None, device: Optional[int] = None,
                 timeout_s: Optional[float] = None, world: Optional[int] = None,
                 rank: Optional[int] = None, unique_id: Optional[bytes] = None):
        import ctypes as C

        from ._lib import lib

        dist = _dist()
        explicit = world is not None
        self.world = world if explicit else (
            dist.get_world_size(group) if dist.is_initialized() else 1)
        self.rank = rank if explicit else (dist.get_rank(group) if dist.is_initialized() else 0)
        uid = (C.c_char * 128)()
        if unique_id is not None:
            C.memmove(uid, unique_id, 128)
        elif self.rank == 0:
            optim._check(lib.mco_comm_unique_id(uid))
        if self.world > 1 and not explicit:
            box = [bytes(uid)]
            src = dist.get_global_rank(group, 0) if group is not None else 0
            dist.broadcast_object_list(box, src=src, group=group)
            C.memmove(uid, box[0], 128)
        h = C.c_void_p()
        self._destroy = lib.mco_comm_destroy
        self.device = optim._device(device)
        optim._check(lib.mco_comm_create_timeout(uid, self.world, self.rank, self.device,
                                                 float(timeout_s or 0.0), C.byref(h)))
        self._h = h

    def wait(self, stream=None) -> None:
        """Host wait for the stream's collectives, bounded by the communicator's deadline
        (ProtocolError naming this rank, communicator aborted, on expiry)."""
        from ._lib import lib

        optim._check(lib.mco_comm_wait(self._h, optim._stream(stream)))

    def abort(self) -> None:
        from ._lib import lib

        optim._check(lib.mco_comm_abort(self._h))

    def allreduce_sum(self, t, stream=None) -> None:
        from ._lib import lib

        optim._check(lib.mco_comm_allreduce_sum(self._h, t.data_ptr(), optim._dtype_code(t),
                                                t.numel(), optim._stream(stream)))

    def check(self) -> None:
        from ._lib import lib

        optim._check(lib.mco_comm_check(self._h))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            self._destroy(h)
            self._h = None


class NativeZeroOptimizer:
    """Stage-2 ZeRO step as one C-ABI call (mco_shard_step): NCCL reduce-scatter of the
    flat gradient -> the sm_100a FlatOptimizer on the ZeroPlan-owned slice -> NCCL
    all-gather of the flat parameters, stream-ordered, no torch collectives.  Same
    ownership and state as ZeroShardedOptimizer (parallel.cpp:656-666)."""

    def __init__(self, cfg: optim.OptimizerConfig, total_len: int, comm: NcclComm,
                 device: Optional[int] = None, mixed: bool = False, master_init=None):
        """mixed: bf16 replicas with an fp32 master of the owned part
        (mco_shard_step_mixed); master_init = the fp32 initial parameters (full vector
        or the owned slice)."""
        self.comm = comm
        self.total_len = int(total_len)
        self.plan = ZeroPlan.make(self.total_len, comm.world, 2)
        self.lo, self.hi = self.plan.owned_range(comm.rank)
        self.opt = optim.FlatOptimizer(cfg, self.hi - self.lo, device=device)
        self.mixed = mixed
        self.master = None
        if mixed:
            if master_init is None:
                raise optim.ContractError("mixed sharding needs the fp32 master init")
            src = master_init if master_init.numel() == self.hi - self.lo else \
                master_init[self.lo:self.hi]
            self._master_src = src.float()

    def step(self, flat_params, flat_grads, lr: float, stream=None) -> None:
        from ._lib import lib

        optim._dev(flat_params, "shard step params")
        optim._dev(flat_grads, "shard step grads")
        if flat_params.numel() != self.total_len or flat_grads.numel() != self.total_len:
            raise optim.ContractError(
                f"shard step: flat buffers of {flat_params.numel()} / {flat_grads.numel()} "
                f"elements for a plan of {self.total_len}")
        if self.mixed:
            if flat_params.dtype.itemsize != 2:
                raise optim.ContractError("mixed shard step: bf16 replicas expected")
            if self.master is None:  # the replica slice's phase, so the step vectorises
                self.master = phased_empty(self.hi - self.lo, self._master_src.dtype,
                                           flat_params.device,
                                           elem_phase(flat_params[self.lo:self.hi]))
                self.master.copy_(self._master_src)
                self._master_src = None
            optim._check(lib.mco_shard_step_mixed(
                self.opt._h, self.comm._h, self.master.data_ptr(), flat_params.data_ptr(),
                flat_grads.data_ptr(), optim._dtype_code(flat_grads), self.total_len,
                float(lr), optim._stream(stream)))
            return
        optim._check(lib.mco_shard_step(self.opt._h, self.comm._h, flat_params.data_ptr(),
                                         optim._dtype_code(flat_params), flat_grads.data_ptr(),
                                         optim._dtype_code(flat_grads), self.total_len,
                                         float(lr), optim._stream(stream)))

    def owned_range(self) -> tuple[int, int]:
        return self.lo, self.hi


class BucketedZeroOptimizer:
    """Bucketed, double-buffered stage-2 ZeRO step over the C-ABI's
    NCCL communicator (mco_zb_*): per bucket of the registry-order flat vector,
    reduce-scatter(SUM) of the bucket's local gradient on the library's comm stream ->
    the fused update of this rank's piece (ZeroPlan within the bucket) -> all-gather of
    the bucket's replicas, issued after the next bucket's reduce-scatter so that
    reduce-scatter overlaps this update (parallel.cpp:656-666, bucketed).

    `step(replicas, flat_grads, lr)`: the whole step from a full local gradient.
    Streaming form (no full-length gradient resident): `begin(replicas, lr)`, then per
    bucket `grad_buffer(k)` (a staging slot, double-buffered) -> fill -> `grad_ready(k)`,
    then `end()`.  replica dtype fp32 (the replicas are the parameters) or bf16 (fp32
    master of the owned pieces, `load_master`)."""

    def __init__(self, cfg: optim.OptimizerConfig, total_len: int, comm: "NcclComm",
                 bucket_elems: int = 0, grad_dtype=None, replica_dtype=None):
        import ctypes as C

        import torch

        from ._lib import lib

        self.comm, self.cfg = comm, cfg
        self.total_len = int(total_len)
        gd = optim.MCO_BF16 if grad_dtype == torch.bfloat16 else optim.MCO_F32
        rd = optim.MCO_BF16 if replica_dtype == torch.bfloat16 else optim.MCO_F32
        self.gdt, self.rdt = gd, rd
        h = C.c_void_p()
        self._destroy = lib.mco_zb_destroy
        optim._check(lib.mco_zb_create(C.byref(cfg._to_c()), comm._h, self.total_len,
                                       int(bucket_elems), gd, rd, C.byref(h)))
        self._h = h
        B, nb, own, fl, ms = C.c_uint64(), C.c_int(), C.c_uint64(), C.c_void_p(), C.c_void_p()
        optim._check(lib.mco_zb_info(h, C.byref(B), C.byref(nb), C.byref(own), C.byref(fl),
                                     C.byref(ms)))
        self.bucket_elems, self.nbuckets, self.owned = B.value, nb.value, own.value
        self._master_ptr = ms.value
        self._fl = C.c_void_p(fl.value)  # the state handle (owned by the mco_zb)
        self.device = comm_device(comm)

    def _flat(self):
        return self._fl

    def pieces(self, rank: Optional[int] = None):
        """[(registry offset, n, state offset)] of `rank`'s pieces in bucket order."""
        import ctypes as C

        from ._lib import lib

        rank = self.comm.rank if rank is None else rank
        out = []
        for k in range(self.nbuckets):
            bo, bl, o, n, so = (C.c_uint64() for _ in range(5))
            optim._check(lib.mco_zb_piece(self._h, k, rank, C.byref(bo), C.byref(bl),
                                          C.byref(o), C.byref(n), C.byref(so)))
            out.append((bo.value + o.value, n.value,
                        so.value if rank == self.comm.rank else None))
        return out

    def master(self):
        if not self._master_ptr:
            return None
        return optim._as_tensor(self._master_ptr, self.owned, optim.MCO_F32, self,
                                self.device)

    def load_master(self, full, stream=None) -> None:
        from ._lib import lib

        optim._check(lib.mco_zb_load_master(self._h, full.data_ptr(), optim._dtype_code(full),
                                            optim._stream(stream)))

    def step(self, replicas, flat_grads, lr: float, stream=None) -> None:
        from ._lib import lib

        optim._dev(replicas, "zb replicas")
        optim._dev(flat_grads, "zb grads")
        if replicas.numel() != self.total_len or flat_grads.numel() != self.total_len:
            raise optim.ContractError(
                f"bucketed shard step: flat buffers of {replicas.numel()} / "
                f"{flat_grads.numel()} elements for a plan of {self.total_len}")
        if optim._dtype_code(replicas) != self.rdt or optim._dtype_code(flat_grads) != self.gdt:
            raise optim.ContractError("bucketed shard step: dtype differs from the plan")
        optim._check(lib.mco_zb_step(self._h, replicas.data_ptr(), flat_grads.data_ptr(),
                                     float(lr), optim._stream(stream)))

    def step_local(self, replicas, flat_grads, lr: float, stream=None) -> None:
        """The same update kernels without the collectives (shard-local cost)."""
        from ._lib import lib

        optim._check(lib.mco_zb_step_local(self._h, replicas.data_ptr(), flat_grads.data_ptr(),
                                           float(lr), optim._stream(stream)))

    def begin(self, replicas, lr: float, stream=None) -> None:
        """replicas=None: ring mode (bf16 replicas only) -- no full replica is resident,
        bucket k is gathered into a two-slot ring (`gathered(k)`)."""
        from ._lib import lib

        if replicas is not None:
            optim._dev(replicas, "zb replicas")
        optim._check(lib.mco_zb_begin(self._h, replicas.data_ptr() if replicas is not None
                                      else None, float(lr), optim._stream(stream)))

    def gathered(self, k: int, stream=None):
        """Ring mode: bucket k's gathered bf16 parameters (valid until bucket k+2's
        update); the stream waits for its all-gather."""
        import ctypes as C

        import torch

        from ._lib import lib

        ptr = C.c_void_p()
        optim._check(lib.mco_zb_gathered(self._h, int(k), C.byref(ptr), optim._stream(stream)))
        n = min(self.bucket_elems, self.total_len - k * self.bucket_elems)
        raw = torch.as_tensor(_U16View(ptr.value, n, self), device=f"cuda:{self.device}")
        return raw.view(torch.bfloat16)

    @staticmethod
    def footprint(kind: int, total_len: int, world: int, bucket_elems: int,
                  replica_dtype_bytes: int = 4, ring: bool = False,
                  grad_dtype_bytes: int = 4) -> dict:
        """Device bytes one rank holds for the bucketed step (the largest rank): fp32
        state of its pieces (kinds' slot counts, optim.cpp:74-98), the fp32 master
        (bf16 replicas), the replicas (or the two ring slots), two gradient staging
        buckets and two reduced pieces."""
        slots = {0: 2, 1: 1, 2: 4, 3: 2}[int(kind)]
        unit = 8 * world
        B = min(bucket_elems or total_len, total_len)
        B = (B + unit - 1) // unit * unit
        nb = (total_len + B - 1) // B
        own = 0
        for k in range(nb):
            L = min(total_len, (k + 1) * B) - k * B
            own += L // world + (1 if L % world else 0)
        out = {"state": slots * own * 4,
               "master": own * 4 if replica_dtype_bytes < 4 else 0,
               "replicas": (2 * B if ring else total_len) * replica_dtype_bytes,
               "staging": 2 * B * grad_dtype_bytes,
               "reduced": 2 * (B // world + 8) * grad_dtype_bytes,
               "owned": own, "bucket_elems": B}
        out["total"] = sum(v for k, v in out.items() if k not in ("owned", "bucket_elems"))
        return out

    def grad_buffer(self, k: int, stream=None):
        import ctypes as C

        import torch

        from ._lib import lib

        ptr, n = C.c_void_p(), C.c_uint64()
        optim._check(lib.mco_zb_grad_buffer(self._h, int(k), C.byref(ptr), C.byref(n),
                                            optim._stream(stream)))
        if self.gdt == optim.MCO_F32:
            return optim._as_tensor(ptr.value, n.value, optim.MCO_F32, self, self.device)
        raw = torch.as_tensor(_U16View(ptr.value, n.value, self),
                              device=f"cuda:{self.device}")
        return raw.view(torch.bfloat16)

    def grad_ready(self, k: int, grad=None, stream=None) -> None:
        from ._lib import lib

        optim._check(lib.mco_zb_grad_ready(self._h, int(k),
                                           grad.data_ptr() if grad is not None else None,
                                           optim._stream(stream)))

    def end(self, stream=None) -> None:
        from ._lib import lib

        optim._check(lib.mco_zb_end(self._h, optim._stream(stream)))

    def steps_taken(self) -> int:
        import ctypes as C

        from ._lib import lib

        t = C.c_int64()
        optim._check(lib.mco_flat_get_steps(self._flat(), C.byref(t)))
        return t.value

    def buffers(self):
        """[(name, device view over this rank's pieces, bucket order)]."""
        import ctypes as C

        from ._lib import lib

        nb = C.c_int()
        optim._check(lib.mco_flat_num_buffers(self._flat(), C.byref(nb)))
        out = []
        for i in range(nb.value):
            name, ptr, ln, dt = C.c_char_p(), C.c_void_p(), C.c_uint64(), C.c_int()
            optim._check(lib.mco_flat_buffer(self._flat(), i, C.byref(name), C.byref(ptr),
                                             C.byref(ln), C.byref(dt)))
            out.append((name.value.decode(),
                        optim._as_tensor(ptr.value, ln.value, dt.value, self, self.device)))
        return out

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            self._destroy(h)
            self._h = None


def comm_device(comm) -> int:
    dev = getattr(comm, "device", None)
    return dev if dev is not None else optim._device(None)
