import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) and the built libaccelgen_b200.so")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        has_cuda = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_cuda = False
    if has_cuda:
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(autouse=True)
def _release_gpu_memory(request):
    """GPU tests build OPT-13B/175B-shaped models, oracle executors on the device and KV pools sized
    from free HBM; hand everything back to the driver between tests so a later test (the TP tests
    spawn one process per rank on the same GPU) sees the whole 180 GB."""
    yield
    if "gpu" not in request.keywords:
        return
    import gc
    import torch
    gc.collect()
    if torch.cuda.is_available():
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        free, total = torch.cuda.mem_get_info()
        if free < 0.6 * total:  # something outlived its test: name it in the log
            print(f"\n[conftest] after {request.node.nodeid}: {free / 2**30:.1f} of {total / 2**30:.1f} GiB free",
                  file=sys.stderr)
