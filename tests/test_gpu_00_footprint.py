"""SURVEY 8(e) C4 at its stated sizes: one rank's device footprint of the bucketed
stage-2 step (zero.BucketedZeroOptimizer.footprint) allocated on one B200 and measured with
cudaMemGetInfo.  Its own file, named to run first among the GPU tests: the check needs
the GPU's memory free, and earlier tests' processes and caches can hold tens of GB
(a 31 GB shortfall was seen late in a full run)."""
import os

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


FOOTPRINT_CHILD = r"""
import gc, json, sys
import torch
sys.path.insert(0, sys.argv[1])
from paper_2312_00407_b200 import optim, registry, zero
from paper_2312_00407_b200.optim import Kind, OptimizerConfig
kind, model, world, ring = {
    "65b-L16 adan mixed N=2": (Kind.ADAN, registry.LLAMA_65B_L16, 2, False),
    "65b sophia ring N=8": (Kind.SOPHIA, registry.LLAMA_65B, 8, True)}[sys.argv[2]]
torch.cuda.set_device(0)
torch.zeros(1, device="cuda")
free0, total = torch.cuda.mem_get_info()
fp = zero.BucketedZeroOptimizer.footprint(kind, model.param_count(), world, 1 << 28, 2, ring)
out = {"fp": fp, "free0": free0, "total": total}
if fp["total"] <= free0 - (1 << 30):
    own, B = fp["owned"], fp["bucket_elems"]
    opt = optim.FlatOptimizer(OptimizerConfig.defaults_for(kind), own)
    bufs = [torch.zeros(own, device="cuda"),
            torch.zeros(fp["replicas"] // 2, dtype=torch.bfloat16, device="cuda"),
            torch.zeros(fp["staging"] // 4, device="cuda"),
            torch.full((fp["reduced"] // 4,), 1e-3, device="cuda")]
    torch.cuda.synchronize()
    out["used"] = free0 - torch.cuda.mem_get_info()[0]
    piece = B // world
    opt.step_mixed(bufs[0][:piece], bufs[3][:piece], bufs[1][:piece], 1e-4)
    torch.cuda.synchronize()
    out["stepped"] = float(bufs[1][:piece].float().abs().max()) > 0
print(json.dumps(out))
"""


@pytest.mark.parametrize("case", ["65b-L16 adan mixed N=2", "65b sophia ring N=8"])
def test_c4_rank_footprint_fits_one_b200(case):
    """SURVEY C4 sizes: one rank's device footprint of the bucketed step
    (BucketedZeroOptimizer.footprint: fp32 state + master of its pieces, bf16 replicas
    or the two ring slots, two staging buckets, two reduced pieces) allocated on one
    B200, measured with cudaMemGetInfo, and a piece updated in it.  65B-L16 Adan with
    full bf16 replicas at N = 2; the full 65B Sophia at N = 8 in ring mode -- its full
    bf16 replicas alone are 130.6 GB and with the 97.9 GB of master + state would not
    fit a 180 GB GPU under stage 1 / 2."""
    import json
    import subprocess
    import sys

    import gc

    gc.collect()
    torch.cuda.empty_cache()
    pfree, ptotal = torch.cuda.mem_get_info()  # what the rest of the GPU holds, for the message
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", FOOTPRINT_CHILD, root, case],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads(r.stdout.strip().splitlines()[-1])
    fp = d["fp"]
    assert fp["total"] < d["total"], d
    assert "used" in d, (f"{case}: {fp['total'] / 1e9:.1f} GB needed, {d['free0'] / 1e9:.1f} GB "
                         f"free in the child ({(ptotal - pfree) / 1e9:.1f} GB in use before it)")
    assert d["stepped"] and fp["total"] * 0.99 <= d["used"] < d["total"], d
    print(f"{case}: {d['used'] / 1e9:.1f} GB per rank of {d['total'] / 1e9:.1f} GB "
          f"({ {k: round(v / 1e9, 2) for k, v in fp.items() if k not in ('owned', 'bucket_elems')} })")

