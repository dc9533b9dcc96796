"""Backward-fused optimizer steps: the reference's
lomo_fused_backward_step / adalomo_fused_step (optim.cpp:284-335) on torch
autograd instead of minicollie's Tape.

Each parameter's update runs in a post-accumulate-grad hook the moment its
gradient is complete (the reference's Tape::add_post_grad_hook, tensor.cpp:215-251),
then the gradient is dropped -- so at most one parameter gradient is alive at a
time plus whatever autograd holds, which is LOMO's memory property
(test_optim.cpp:286-316).  The update itself is the sm_100a kernel behind the C-ABI
(lomo_apply / lomo_apply_clipped / AdaLomoState.apply); with a process group the
hook first all-reduces (SUM) the gradient, as the reference's fused DP path does
(parallel.cpp:585-599).
"""
from __future__ import annotations

from typing import Callable, Optional, Sequence

from . import optim


def _hooks(params, fn):
    handles = [p.register_post_accumulate_grad_hook(fn) for p in params]
    return handles


def _dp_reduce(p, group):
    if group is None:
        return
    import torch.distributed as dist

    if dist.get_world_size(group) > 1:
        dist.all_reduce(p.grad, op=dist.ReduceOp.SUM, group=group)


def lomo_fused_backward_step(params: Sequence, loss_fn: Callable, lr: float,
                             clip_norm: Optional[float] = None, group=None):
    """optim.cpp:284-318.  With clip_norm: pass 1 accumulates the global sum of
    squares of every gradient on the device (deterministic kernel) and drops each
    gradient at once; pass 2 re-runs forward + backward and applies
    p -= lr * scale * g per parameter with scale = clip/||g|| iff ||g|| > clip.
    Returns the loss value of the update pass."""
    import torch

    params = list(params)
    norm2 = None
    if clip_norm is not None:
        norm2 = torch.zeros((), dtype=torch.float64, device=params[0].device)

        def acc(p):
            _dp_reduce(p, group)
            optim.sumsq(p.grad, out=norm2, accumulate=True)
            p.grad = None

        hs = _hooks(params, acc)
        try:
            loss_fn().backward()
        finally:
            for h in hs:
                h.remove()

    def upd(p):
        _dp_reduce(p, group)
        with torch.no_grad():
            if norm2 is None:
                optim.lomo_apply(p.data, p.grad, lr, 1.0)
            else:
                optim.lomo_apply_clipped(p.data, p.grad, lr, norm2, clip_norm)
        p.grad = None

    hs = _hooks(params, upd)
    try:
        loss = loss_fn()
        value = loss.detach()
        loss.backward()
    finally:
        for h in hs:
            h.remove()
    return value


def adalomo_fused_step(params: Sequence, loss_fn: Callable, lr: float,
                       state: "optim.AdaLomoState", group=None):
    """optim.cpp:320-335: AdaLomoState::apply per parameter inside backward.
    `state` was created with the parameters' shapes in the same order."""
    import torch

    params = list(params)
    index = {id(p): k for k, p in enumerate(params)}

    def upd(p):
        _dp_reduce(p, group)
        with torch.no_grad():
            state.apply(index[id(p)], p.data, p.grad, lr)
        p.grad = None

    hs = _hooks(params, upd)
    try:
        loss = loss_fn()
        value = loss.detach()
        loss.backward()
    finally:
        for h in hs:
            h.remove()
    return value
