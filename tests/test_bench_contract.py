"""The bench.py JSON contract for the reference arm (runs on CPU: the compiled
reference on the host cores).  The GPU arm is exercised on the B200 box."""
import json
import os
import subprocess
import sys

import pytest

import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(O.ref is None, reason="oracle/_ref not built")
def test_reference_arm_prints_one_contract_line():
    env = dict(os.environ, MCO_CPU_SAMPLE="tiny")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--steps", "1", "--warmup", "1"], capture_output=True, text=True,
                       env=env, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "cpu_baseline", "e2e", "impl"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert set(d["per_optimizer"]) == {"adamw", "lion", "adan", "sophia", "lomo", "adalomo"}
    assert d["config"]["params"] == 2 * (4 * 256 * 256 + 3 * 256 * 688 + 2 * 256)


@pytest.mark.skipif(O.ref is None, reason="oracle/_ref not built")
def test_reference_arm_loads_no_product_code():
    """The reference arm runs only the compiled reference: neither the product package
    nor libmco.so is loaded in its process."""
    code = ("import os, sys, bench; "
            "os.environ['MCO_CPU_SAMPLE'] = 'tiny'; "
            "bench.run_cpu_reference(0, 1); bench.run_cpu_single_thread(); "
            "maps = open('/proc/self/maps').read(); "
            "assert 'paper_2312_00407_b200' not in sys.modules, 'package imported'; "
            "assert 'libmco.so' not in maps, 'libmco.so mapped'; "
            "assert 'libmco_ref.so' in maps; print('clean')")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                       timeout=600, cwd=ROOT)
    assert r.returncode == 0 and "clean" in r.stdout, r.stderr[-2000:]


@pytest.mark.skipif(O.ref is None, reason="oracle/_ref not built")
def test_gpus_flag_launches_that_many_ranks():
    """`python bench.py --gpus 2` (no torchrun) re-launches itself with 2 ranks; the
    line reports n_gpus == 2 (the reference arm: rank 0 alone prints)."""
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["MCO_CPU_SAMPLE"] = "tiny"
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--gpus", "2", "--steps", "1", "--warmup", "0"], capture_output=True,
                       text=True, env=env, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong"


def test_gpus_flag_disagreeing_with_world_size_is_an_error():
    env = dict(os.environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "4"],
                       capture_output=True, text=True, env=env, timeout=300, cwd=ROOT)
    assert r.returncode == 2 and "WORLD_SIZE=2" in r.stderr
