"""Bucketed, backward-overlapped ZeRO step on CPU with gloo, world
size 2 and 3: gradients accumulate into the flat buffer, each bucket is reduced to
its ZeroPlan owners, stepped and broadcast from inside backward, and the result is
the serial FlatOptimizer step on the rank-summed gradient (SerialBaseline,
tests/serial_ref.hpp:34-70).  The per-piece update is the oracle here (no GPU)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
STEPS = 3
LR = 1e-2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


class Net(torch.nn.Module):
    """Three layers plus one parameter the loss never touches (its bucket is flushed
    by finish() with a zero gradient)."""

    def __init__(self):
        super().__init__()
        g = torch.Generator().manual_seed(11)
        self.l1 = torch.nn.Linear(8, 16).double()
        self.l2 = torch.nn.Linear(16, 12).double()
        self.l3 = torch.nn.Linear(12, 4).double()
        self.unused = torch.nn.Parameter(torch.zeros(5, dtype=torch.float64))
        with torch.no_grad():
            for p in self.parameters():
                p.copy_(torch.randn(p.shape, generator=g, dtype=torch.float64) * 0.3)

    def forward(self, x):
        return self.l3(torch.tanh(self.l2(torch.tanh(self.l1(x)))))


def _data(rank, t):
    g = torch.Generator().manual_seed(1000 * rank + t)
    return (torch.randn(6, 8, generator=g, dtype=torch.float64),
            torch.randn(6, 4, generator=g, dtype=torch.float64))


def _loss(net, rank, t):
    x, y = _data(rank, t)
    return ((net(x) - y) ** 2).mean()


def _worker(rank, world, kind, bucket, port, out_q):
    import sys

    for p in (ROOT, os.path.join(ROOT, "oracle")):
        sys.path.insert(0, p)
    import oracle as O
    from paper_2312_00407_b200 import overlap
    from paper_2312_00407_b200.optim import OptimizerConfig

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = OptimizerConfig.defaults_for(kind)
        cfg.weight_decay = 0.01
        orcs = {}

        def local(p, g, lr, piece):
            if piece not in orcs:
                orcs[piece] = O.OracleFlat(cfg, p.numel(), np.float64)
            orcs[piece].step(p.numpy(), np.ascontiguousarray(g.numpy()), lr)

        net = Net()
        opt = overlap.OverlappedZeroOptimizer(cfg, list(net.parameters()), bucket_elems=bucket,
                                              local_step=local)
        in_bw = []
        for t in range(1, STEPS + 1):
            opt.backward_step(lambda: _loss(net, rank, t), LR)
            assert opt.launch_log == list(range(len(opt.buckets)))
            in_bw.append(opt.launched_in_backward)
        flat = opt.flat_params.numpy().copy()
        # the module's own parameters ARE the flat buffer (zero-copy)
        cat = torch.cat([p.detach().reshape(-1) for p in net.parameters()]).numpy()
        assert np.array_equal(cat, flat)
        state = {}
        for name in orcs[next(iter(orcs))].state:
            state[name] = np.concatenate([orcs[k].state[name] for k in sorted(orcs)])
        out_q.put((rank, {"flat": flat, "range": opt.owned_range(), "state": state,
                          "nbuckets": len(opt.buckets), "in_backward": in_bw}))
    finally:
        dist.destroy_process_group()


def _run(world, kind, bucket):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, kind, bucket, port, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


def _serial(world, kind):
    import oracle as O
    from paper_2312_00407_b200.optim import OptimizerConfig

    cfg = OptimizerConfig.defaults_for(kind)
    cfg.weight_decay = 0.01
    net = Net()
    params = list(net.parameters())
    flat = torch.cat([p.detach().reshape(-1) for p in params]).numpy().copy()
    orc = O.OracleFlat(cfg, flat.size, np.float64)
    for t in range(1, STEPS + 1):
        gsum = None
        for r in range(world):
            with torch.no_grad():
                off = 0
                for p in params:
                    p.copy_(torch.from_numpy(flat[off:off + p.numel()]).view_as(p))
                    off += p.numel()
            for p in params:
                p.grad = None
            _loss(net, r, t).backward()
            g = torch.cat([(p.grad if p.grad is not None else torch.zeros_like(p)).reshape(-1)
                           for p in params]).numpy()
            gsum = g.copy() if gsum is None else gsum + g
        orc.step(flat, gsum, LR)
    return flat, orc.state


@pytest.mark.parametrize("world,kind,bucket", [(2, 0, 150), (2, 2, 64), (3, 3, 100),
                                               (3, 1, 1 << 20)])
def test_overlapped_step_equals_serial(world, kind, bucket):
    res = _run(world, kind, bucket)
    want, want_state = _serial(world, kind)
    ranges = [res[r]["range"] for r in range(world)]
    assert ranges[0][0] == 0 and ranges[-1][1] == want.size
    for r in range(world):
        got = res[r]["flat"]
        if world == 2:
            assert np.array_equal(got, want)  # a + b: exact
        else:
            np.testing.assert_allclose(got, want, rtol=1e-13, atol=1e-16)
        lo, hi = ranges[r]
        for name, buf in res[r]["state"].items():
            np.testing.assert_allclose(buf, want_state[name][lo:hi], rtol=1e-12, atol=1e-300)
        nb = res[r]["nbuckets"]
        if nb > 1:  # all but the bucket holding the unused parameter launch mid-backward
            assert all(x == nb - 1 for x in res[r]["in_backward"]), res[r]["in_backward"]
