import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a kernels)")
    config.addinivalue_line("markers", "multigpu: needs >= 2 GPUs (device-flag paths)")


def _ngpu() -> int:
    try:
        import torch
        return torch.cuda.device_count() if torch.cuda.is_available() else 0
    except Exception:
        return 0


NGPU = _ngpu()


def pytest_collection_modifyitems(config, items):
    skip_gpu = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords and NGPU == 0:
            item.add_marker(skip_gpu)


def need_gpus(n: int):
    return pytest.mark.skipif(NGPU < n, reason=f"needs {n} GPUs, have {NGPU}")
