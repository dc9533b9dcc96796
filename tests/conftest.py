import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def _has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


def pytest_collection_modifyitems(config, items):
    if _has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


def pytest_runtest_teardown(item, nextitem):
    """MCO_MEMLOG=path: device memory in use after every GPU test (leak hunting)."""
    path = os.environ.get("MCO_MEMLOG")
    if not path or "gpu" not in item.keywords or not _has_gpu():
        return
    import gc

    import torch
    gc.collect()
    torch.cuda.empty_cache()
    free, total = torch.cuda.mem_get_info()
    with open(path, "a") as f:
        f.write(f"{(total - free) / 1e9:.2f} GB {item.nodeid}\n")
