"""Backward-fused optimizer steps: the reference's
lomo_fused_backward_step / adalomo_fused_step (optim.cpp:284-335) on torch
autograd instead of minicollie's Tape.

Each parameter's update runs in a post-accumulate-grad hook the moment its
gradient is complete (the reference's Tape::add_post_grad_hook, tensor.cpp:215-251),
then the gradient is dropped -- so at most one parameter gradient is alive at a
time plus whatever autograd holds, which is LOMO's memory property
(test_optim.cpp:286-316).  The update itself is the sm_100a kernel behind the C-ABI
(lomo_apply / lomo_apply_clipped / AdaLomoState.apply).

With a process group the gradient is SUM-all-reduced first, as the reference's fused
DP path does (parallel.cpp:585-599): one all-reduce per parameter (the reference's
behaviour), or -- with ``bucket_elems`` -- gradients are packed into one reusable flat
bucket and all-reduced together, then every packed parameter is updated from its
view of the reduced bucket (a bucketed DP all-reduce instead of one
per parameter, parallel.cpp:591).  Live gradient memory stays bounded by the bucket
plus one tensor.
"""
from __future__ import annotations

from typing import Callable, Optional, Sequence

from . import optim


class _CudaOps:
    sumsq = staticmethod(optim.sumsq)
    lomo_apply = staticmethod(optim.lomo_apply)
    lomo_apply_clipped = staticmethod(optim.lomo_apply_clipped)
    lomo_apply_list = staticmethod(optim.lomo_apply_list)


def _hooks(params, fn):
    handles = [p.register_post_accumulate_grad_hook(fn) for p in params]
    return handles


def _world(group) -> int:
    if group is None:
        return 1
    import torch.distributed as dist

    return dist.get_world_size(group)


class _GradPath:
    """Delivers each parameter's (DP-reduced) gradient to ``fn(p, grad)``.

    Unbucketed: all_reduce(p.grad) per parameter (parallel.cpp:591), then fn.
    Bucketed: p.grad is copied into a flat bucket and dropped; when the next gradient
    would not fit (or at flush), the bucket is all-reduced once and fn runs for every
    packed parameter on its view.  A gradient larger than the bucket is reduced alone.
    """

    def __init__(self, fn: Callable, group, bucket_elems: Optional[int],
                 group_fn: Optional[Callable] = None):
        self.fn, self.group, self.group_fn = fn, group, group_fn
        self.bucket_elems = bucket_elems or None
        self.world = _world(group)
        self.buf = None
        self.items: list = []
        self.used = 0

    def _allreduce(self, t) -> None:
        if self.world == 1:
            return
        import torch.distributed as dist

        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)

    def add(self, p) -> None:
        import torch

        if self.bucket_elems is None:
            self._allreduce(p.grad)
            self.fn(p, p.grad)
            p.grad = None
            return
        n = p.grad.numel()
        if n > self.bucket_elems:  # oversize: reduce alone, keep the order of updates
            self.flush()
            self._allreduce(p.grad)
            self.fn(p, p.grad)
            p.grad = None
            return
        if self.buf is None or self.buf.dtype != p.grad.dtype or self.buf.device != p.grad.device:
            self.flush()
            # zeros: the alignment gaps below only ever hold finite values
            self.buf = torch.zeros(self.bucket_elems, dtype=p.grad.dtype, device=p.grad.device)
        # every packed gradient starts on the 8-element grid, as a separately allocated
        # gradient would: the update kernels take their vector path for it, and the
        # result equals the per-parameter path bit for bit
        start = (self.used + 7) // 8 * 8
        if start + n > self.bucket_elems:
            self.flush()
            start = 0
        self.buf[start:start + n].copy_(p.grad.reshape(-1))
        self.items.append((p, start, n))
        self.used = start + n
        p.grad = None

    def flush(self) -> None:
        if not self.items:
            return
        self._allreduce(self.buf[:self.used])
        views = [(p, self.buf[off:off + n].view_as(p)) for p, off, n in self.items]
        if self.group_fn is not None:
            self.group_fn(views)  # the whole bucket in one call (list forms)
        else:
            for p, g in views:
                self.fn(p, g)
        self.items, self.used = [], 0


def _run_backward(params, grad_fn, loss_fn, group, bucket_elems, want_loss, group_fn=None):
    path = _GradPath(grad_fn, group, bucket_elems, group_fn)
    hs = _hooks(params, lambda p: path.add(p))
    try:
        loss = loss_fn()
        value = loss.detach() if want_loss else None
        loss.backward()
        path.flush()
    finally:
        for h in hs:
            h.remove()
    return value


def lomo_fused_backward_step(params: Sequence, loss_fn: Callable, lr: float,
                             clip_norm: Optional[float] = None, group=None,
                             bucket_elems: Optional[int] = None, ops=_CudaOps):
    """optim.cpp:284-318.  With clip_norm: pass 1 accumulates the global sum of
    squares of every (reduced) gradient on the device (deterministic kernel) and drops
    each gradient at once; pass 2 re-runs forward + backward and applies
    p -= lr * scale * g per parameter with scale = clip/||g|| iff ||g|| > clip.
    Returns the loss value of the update pass.  ``ops`` is the kernel set (CUDA by
    default; the CPU tests inject the oracle)."""
    import torch

    params = list(params)
    norm2 = None
    if clip_norm is not None:
        norm2 = torch.zeros((), dtype=torch.float64, device=params[0].device)

        def acc(p, g):
            ops.sumsq(g, out=norm2, accumulate=True)

        _run_backward(params, acc, loss_fn, group, bucket_elems, False)

    def upd(p, g):
        with torch.no_grad():
            if norm2 is None:
                ops.lomo_apply(p.data, g, lr, 1.0)
            else:
                ops.lomo_apply_clipped(p.data, g, lr, norm2, clip_norm)

    def upd_bucket(views):  # the whole bucket in one launch (mco_lomo_apply_list)
        with torch.no_grad():
            ops.lomo_apply_list([p.data for p, _ in views], [g for _, g in views], lr, 1.0,
                                norm2, clip_norm if norm2 is not None else None)

    group_fn = upd_bucket if bucket_elems and hasattr(ops, "lomo_apply_list") else None
    return _run_backward(params, upd, loss_fn, group, bucket_elems, True, group_fn=group_fn)


def adalomo_fused_step(params: Sequence, loss_fn: Callable, lr: float,
                       state: "optim.AdaLomoState", group=None,
                       bucket_elems: Optional[int] = None):
    """optim.cpp:320-335: AdaLomoState::apply per parameter inside backward.
    `state` was created with the parameters' shapes in the same order."""
    import torch

    params = list(params)
    index = {id(p): k for k, p in enumerate(params)}

    def upd(p, g):
        with torch.no_grad():
            state.apply(index[id(p)], p.data, g.contiguous(), lr)

    def upd_bucket(views):
        # runs of consecutive registry indices -> one list call each (mco_adalomo_apply_list)
        views = sorted(views, key=lambda pg: index[id(pg[0])])
        run = [views[0]]
        for pg in views[1:] + [None]:
            if pg is not None and index[id(pg[0])] == index[id(run[-1][0])] + 1:
                run.append(pg)
                continue
            with torch.no_grad():
                state.apply_list(index[id(run[0][0])], [p.data for p, _ in run],
                                 [g.contiguous() for _, g in run], lr)
            if pg is not None:
                run = [pg]

    return _run_backward(params, upd, loss_fn, group, bucket_elems, True,
                         group_fn=upd_bucket if bucket_elems else None)
