import os
import sys

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")


import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (sm_100a) device")


def pytest_collection_modifyitems(config, items):
    try:
        import torch

        has_gpu = torch.cuda.is_available()
    except Exception:  # noqa: BLE001
        has_gpu = False
    if has_gpu:
        if any("gpu" in item.keywords for item in items):
            _warm_torch_kernels()
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


def _warm_torch_kernels():
    """Load the torch kernels that rank bodies launch (casts, copies, clamp,
    fills, matmul, comparisons) before any test: under lazy module loading
    the first launch of a kernel synchronises the context, and inside a rank
    body that would wait for a sibling rank's spinning fused kernel on the
    same GPU."""
    import torch

    x = torch.randn(256, 256, device="cuda")
    xb = x.bfloat16()
    h = torch.from_numpy(np.ones((64, 64))).to(torch.bfloat16).to("cuda")
    y = (xb @ xb).float() + torch.clamp(xb, -2, 2).float()
    y.fill_(float("nan"))
    torch.equal(xb.view(torch.int16), xb.view(torch.int16))
    (x - xb.float()).norm() / x.norm()
    torch.zeros(8, device="cuda", dtype=torch.int64).sum()
    torch.clamp(h, -2, 2).half().float().cpu()
    torch.cuda.synchronize()


@pytest.fixture
def rng():
    return np.random.default_rng(1234)
