import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

REFERENCE_SRC = Path("/root/reference/pkg/src")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device")
    config.addinivalue_line("markers", "slow: long-running")


def have_cuda() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def reference():
    """The live reference package (only in the build container)."""
    if not REFERENCE_SRC.exists():
        pytest.skip("reference not mounted")
    if str(REFERENCE_SRC) not in sys.path:
        sys.path.insert(0, str(REFERENCE_SRC))
    os.environ.setdefault("BAYERMC_THREADS", "1")
    import bayermc.fme  # noqa: F401
    import bayermc.frame_select  # noqa: F401
    import bayermc.mv_refine  # noqa: F401
    import bayermc.pipeline  # noqa: F401
    import bayermc.propagate  # noqa: F401
    import bayermc
    return bayermc


@pytest.fixture(scope="session")
def cuda():
    # gpu-marked tests must never pass silently without the device
    if not have_cuda():
        pytest.fail("gpu test selected but no CUDA device is visible")
    import torch
    return torch
