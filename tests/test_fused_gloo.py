"""Backward-fused LOMO with data parallelism on CPU (gloo, world size 2): the
reference's per-parameter gradient all-reduce inside the hook (parallel.cpp:585-599)
and the bucketed all-reduce give the serial result -- SGD on the
rank-summed gradient, with the global-norm clip computed on the summed gradient.
The kernels are replaced by CPU restatements here (no GPU); tests/test_gpu_fused_backward.py
runs the CUDA path."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


class CpuOps:
    @staticmethod
    def sumsq(g, out=None, accumulate=False, stream=None):
        v = (g.double() ** 2).sum()
        out.add_(v) if accumulate else out.copy_(v)
        return out

    @staticmethod
    def lomo_apply(p, g, lr, scale, stream=None):
        p.sub_((lr * scale) * g)

    @staticmethod
    def lomo_apply_clipped(p, g, lr, s, clip, stream=None):
        norm = float(s.item()) ** 0.5
        scale = clip / norm if (norm > clip and norm > 0) else 1.0
        p.sub_((lr * scale) * g)


def make_net():
    g = torch.Generator().manual_seed(5)
    net = torch.nn.Sequential(torch.nn.Linear(6, 20), torch.nn.Tanh(), torch.nn.Linear(20, 9),
                              torch.nn.Tanh(), torch.nn.Linear(9, 3)).double()
    with torch.no_grad():
        for p in net.parameters():
            p.copy_(torch.randn(p.shape, generator=g, dtype=torch.float64) * 0.4)
    return net


def loss_of(net, rank, t):
    g = torch.Generator().manual_seed(100 * rank + t)
    x = torch.randn(5, 6, generator=g, dtype=torch.float64)
    y = torch.randn(5, 3, generator=g, dtype=torch.float64)
    return ((net(x) - y) ** 2).mean()


CASES = [(None, None), (None, 64), (0.05, None), (0.05, 64), (0.05, 10)]


def _worker(rank, world, port, out_q):
    import sys

    sys.path.insert(0, ROOT)
    from paper_2312_00407_b200 import fused

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = {}
        for clip, bucket in CASES:
            net = make_net()
            for t in range(1, 4):
                fused.lomo_fused_backward_step(list(net.parameters()),
                                               lambda: loss_of(net, rank, t), 0.1,
                                               clip_norm=clip, group=dist.group.WORLD,
                                               bucket_elems=bucket, ops=CpuOps)
            assert all(p.grad is None for p in net.parameters())
            res[(clip, bucket)] = torch.cat(
                [p.detach().reshape(-1) for p in net.parameters()]).numpy().copy()
        # numpy, not tensors: a tensor in a Queue is passed by file descriptor, which
        # races with this process's exit
        out_q.put((rank, res))
    finally:
        dist.destroy_process_group()


def _serial(world, clip):
    net = make_net()
    params = list(net.parameters())
    for t in range(1, 4):
        gs = []
        for r in range(world):
            for p in params:
                p.grad = None
            loss_of(net, r, t).backward()
            gs.append([p.grad.clone() for p in params])
        g = [gs[0][k] + gs[1][k] for k in range(len(params))]
        scale = 1.0
        if clip is not None:
            norm = float(sum((x.double() ** 2).sum() for x in g)) ** 0.5
            scale = clip / norm if norm > clip else 1.0
        with torch.no_grad():
            for p, x in zip(params, g):
                p.sub_((0.1 * scale) * x)
    return torch.cat([p.detach().reshape(-1) for p in params])


def test_fused_lomo_dp_per_parameter_and_bucketed_equal_serial():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res = {r: {k: torch.from_numpy(v) for k, v in d.items()} for r, d in res.items()}
    for clip, bucket in CASES:
        want = _serial(2, clip)
        for r in range(2):
            got = res[r][(clip, bucket)]
            if clip is None:  # a + b is exact
                assert torch.equal(got, want), (bucket, float((got - want).abs().max()))
            else:  # the serial sum of squares runs in registry order, the hooks in
                # backward order: the clip scale may differ in its last bit
                torch.testing.assert_close(got, want, rtol=1e-14, atol=1e-16)
            # bucketing changes neither the reduction nor the order of the updates
            assert torch.equal(got, res[r][(clip, None)])
            assert torch.equal(got, res[1 - r][(clip, bucket)])
