"""Gradient path feeding the sharded optimizer, overlapped with backward.

Reference: ParallelWorker::train_step runs backward, then flattens every parameter
gradient into one vector (parallel.cpp:468-494), reduces it through the hub
(stage 2: reduce-scatter, parallel.cpp:656-658), steps the owned slice
(parallel.cpp:660), all-gathers the parameters (parallel.cpp:661-663) and scatters
them back into the tensors.  Every step is serial after backward.

Here the same step is fed straight from backward:

* zero-copy flat buffers -- each parameter's ``.data`` and ``.grad`` are views of two
  flat buffers in registry order, so autograd accumulates directly into the flat
  gradient and the update writes the parameters in place (no flatten / scatter);
* buckets -- runs of consecutive parameters in REVERSE registry order (the order in
  which backward completes them), each one contiguous range of the flat buffers;
* as soon as a bucket's last gradient is accumulated (post-accumulate-grad hook), a
  side stream runs, for every ZeroPlan piece of the bucket: reduce(SUM) of the
  gradient piece to its owner -> the owner's FlatOptimizer step on that piece (the
  sm_100a kernel) -> broadcast of the piece's new parameters.  Backward keeps running
  on the compute stream meanwhile; ``finish()`` joins the two streams.

Ownership is ZeroPlan over the whole flat vector (parallel.cpp:20-38), so the state a
rank holds is exactly ZeroShardedOptimizer's; ``extract_state()`` returns it by name
(parallel.cpp:820-862).  The result equals the serial FlatOptimizer step on the
rank-summed gradient (SerialBaseline, tests/serial_ref.hpp:34-70).  Buckets are
launched in index order on every rank, as collectives must match across ranks.
An AccumulateGrad node runs once per backward (the engine sums every contribution to
a leaf first), and every node that reads a weight produces that weight's gradient, so
a bucket is complete only after backward has finished reading its parameters.
"""
from __future__ import annotations

from typing import Callable, Optional, Sequence

from . import optim
from .zero import ZeroPlan, _dist, check_agreement


class OverlappedZeroOptimizer:
    """ZeRO stage-2 step on bucketed gradients, launched from inside backward.

    params:       the model's parameters in registry order (rebound to flat views).
    bucket_elems: minimum elements per bucket (a bucket closes at a parameter boundary).
    local_step:   optional ``f(p_piece, g_piece, lr, piece_id)`` replacing the CUDA
                  FlatOptimizer (the CPU tests inject the oracle, as for ZeroShardedOptimizer).
    """

    def __init__(self, cfg: optim.OptimizerConfig, params: Sequence, group=None,
                 bucket_elems: int = 1 << 24, local_step: Optional[Callable] = None):
        import torch

        dist = _dist()
        self.cfg = cfg
        self.params = list(params)
        if not self.params:
            raise optim.ContractError("OverlappedZeroOptimizer: no parameters")
        dev, dtype = self.params[0].device, self.params[0].dtype
        if any(p.device != dev or p.dtype != dtype for p in self.params):
            raise optim.ContractError("OverlappedZeroOptimizer: mixed devices / dtypes")
        self.device = dev
        sizes = [p.numel() for p in self.params]
        self.offsets = [0]
        for n in sizes:
            self.offsets.append(self.offsets[-1] + n)
        P = self.offsets[-1]

        # zero-copy flat buffers (removes parallel.cpp:468-494)
        self.flat_params = torch.empty(P, dtype=dtype, device=dev)
        self.flat_grads = torch.zeros(P, dtype=dtype, device=dev)
        with torch.no_grad():
            for k, p in enumerate(self.params):
                a, b = self.offsets[k], self.offsets[k + 1]
                self.flat_params[a:b].copy_(p.detach().reshape(-1))
                p.data = self.flat_params[a:b].view_as(p)
                p.grad = self.flat_grads[a:b].view_as(p)

        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        check_agreement("OverlappedZeroOptimizer",
                        dict(shapes=[tuple(p.shape) for p in self.params],
                             bucket_elems=bucket_elems, kind=int(cfg.kind)), group)
        self.plan = ZeroPlan.make(P, self.world, 2)
        self.lo, self.hi = self.plan.owned_range(self.rank)

        # buckets in reverse registry order; pieces = bucket range x ZeroPlan parts
        self.buckets: list[list[int]] = []
        cur, cur_n = [], 0
        for k in reversed(range(len(self.params))):
            cur.append(k)
            cur_n += sizes[k]
            if cur_n >= bucket_elems:
                self.buckets.append(cur)
                cur, cur_n = [], 0
        if cur:
            self.buckets.append(cur)
        self.bucket_of = {k: i for i, ks in enumerate(self.buckets) for k in ks}
        self.pieces: list[list[tuple[int, int, int]]] = []  # per bucket: (owner, a, b)
        for ks in self.buckets:
            a, b = self.offsets[min(ks)], self.offsets[max(ks) + 1]
            ps = []
            for r in range(self.world):
                lo, hi = self.plan.owned_range(r)
                x, y = max(a, lo), min(b, hi)
                if x < y:
                    ps.append((r, x, y))
            self.pieces.append(ps)

        # one FlatOptimizer per owned piece; every piece steps once per step, so the
        # step counters stay equal (checked in extract_state)
        self._local = local_step
        self._opt: dict[tuple[int, int], optim.FlatOptimizer] = {}
        if local_step is None:
            for ps in self.pieces:
                for r, a, b in ps:
                    if r == self.rank:
                        self._opt[(a, b)] = optim.FlatOptimizer(cfg, b - a, device=dev.index)
        # high-priority side stream: bucket updates are scheduled ahead of queued backward
        # CTAs, so they overlap instead of waiting for a gap in the compute stream
        self._side = torch.cuda.Stream(dev, priority=-1) if dev.type == "cuda" else None
        self._ready = [0] * len(self.buckets)
        self._next = 0
        self._lr = None
        self._handles = [p.register_post_accumulate_grad_hook(self._hook(k))
                         for k, p in enumerate(self.params)]
        self.launch_log: list[int] = []  # bucket indices in launch order (tests)
        self.launched_in_backward = 0     # buckets launched from hooks, i.e. mid-backward
        self.bucket_events: list = []     # CUDA event after each bucket's side-stream work

    # ---- step protocol --------------------------------------------------------------
    def begin(self, lr: float) -> None:
        """Arm the hooks for one step: zero the flat gradient (after the previous
        step's side-stream work) and reset the bucket counters."""
        import torch

        if self._side is not None:
            torch.cuda.current_stream(self.device).wait_stream(self._side)
        self.flat_grads.zero_()
        esz = self.flat_grads.element_size()
        for k, p in enumerate(self.params):  # someone may have dropped / replaced a .grad
            want = self.flat_grads.data_ptr() + self.offsets[k] * esz
            if p.grad is None or p.grad.data_ptr() != want:
                p.grad = self.flat_grads[self.offsets[k]:self.offsets[k + 1]].view_as(p)
        self._ready = [0] * len(self.buckets)
        self._next = 0
        self._lr = float(lr)
        self.launch_log = []
        self.launched_in_backward = 0
        self.bucket_events = []

    def finish(self) -> None:
        """Launch the buckets whose gradients never arrived (unused parameters: zero
        gradient), in order, and make the compute stream wait for the side stream."""
        import torch

        if self._lr is None:
            raise optim.ContractError("OverlappedZeroOptimizer.finish without begin")
        while self._next < len(self.buckets):
            self._run_bucket(self._next)
            self._next += 1
        if self._side is not None:
            torch.cuda.current_stream(self.device).wait_stream(self._side)
        self._lr = None

    def backward_step(self, loss_fn: Callable, lr: float):
        """begin -> forward -> backward (buckets reduce / step / broadcast as they
        complete) -> finish.  Returns the loss value (detached)."""
        self.begin(lr)
        loss = loss_fn()
        value = loss.detach()
        loss.backward()
        self.finish()
        return value

    # ---- internals ------------------------------------------------------------------
    def _hook(self, k: int):
        def fn(_p):
            if self._lr is None:
                return  # not armed: a plain backward outside a step
            b = self.bucket_of[k]
            self._ready[b] += 1
            while (self._next < len(self.buckets)
                   and self._ready[self._next] == len(self.buckets[self._next])):
                self._run_bucket(self._next)
                self._next += 1
                self.launched_in_backward += 1
        return fn

    def _run_bucket(self, i: int) -> None:
        import contextlib

        import torch

        dist = _dist()
        self.launch_log.append(i)
        ctx = contextlib.nullcontext()
        if self._side is not None:
            self._side.wait_stream(torch.cuda.current_stream(self.device))
            ctx = torch.cuda.stream(self._side)
        with ctx, torch.no_grad():
            pieces = self.pieces[i]
            if self.world > 1:
                for r, a, b in pieces:  # RS of this bucket = reduce to each piece's owner
                    dist.reduce(self.flat_grads[a:b], dst=self._global(r),
                                op=dist.ReduceOp.SUM, group=self.group)
            for r, a, b in pieces:
                if r != self.rank:
                    continue
                p, g = self.flat_params[a:b], self.flat_grads[a:b]
                if self._local is not None:
                    self._local(p, g, self._lr, (a, b))
                else:
                    self._opt[(a, b)].step(p, g, self._lr)
            if self.world > 1:
                for r, a, b in pieces:  # AG of this bucket = broadcast from each owner
                    dist.broadcast(self.flat_params[a:b], src=self._global(r),
                                   group=self.group)
            if self._side is not None:  # completion marker (overlap evidence)
                ev = torch.cuda.Event(enable_timing=True)
                ev.record(self._side)
                self.bucket_events.append(ev)

    def _global(self, r: int) -> int:
        return _dist().get_global_rank(self.group, r) if self.group is not None else r

    # ---- checkpoint hand-off (parallel.cpp:820-862) ----------------------------------
    def owned_range(self) -> tuple[int, int]:
        return self.lo, self.hi

    def extract_state(self) -> dict:
        """The owned slice's named buffers (pieces concatenated in flat order) and t --
        the same layout ZeroShardedOptimizer.extract_state returns."""
        import torch

        out = {"steps": 0, "buffers": {}}
        if not self._opt:
            return out
        keys = sorted(self._opt)
        steps = {self._opt[k].steps_taken() for k in keys}
        if len(steps) != 1:
            raise optim.ProtocolError(f"bucket optimizers out of step: {sorted(steps)}")
        out["steps"] = steps.pop()
        names = [n for n, _ in self._opt[keys[0]].buffers()]
        for name in names:
            out["buffers"][name] = torch.cat(
                [dict(self._opt[k].buffers())[name] for k in keys]).clone()
        return out

    def load_state(self, state: dict) -> None:
        for (a, b), opt in self._opt.items():
            for name, t in opt.buffers():
                src = state["buffers"].get(name)
                if src is not None and src.numel() == self.hi - self.lo:
                    t.copy_(src[a - self.lo:b - self.lo])
            opt.set_steps_taken(state["steps"])

    def state_bytes_runtime(self) -> int:
        return sum(o.state_bytes_runtime() for o in self._opt.values())

    def remove_hooks(self) -> None:
        for h in self._handles:
            h.remove()
        self._handles = []
