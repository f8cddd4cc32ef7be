import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

# The reference simulator is importable only in the build container (it is
# not shipped to the GPU box); tests that need it skip elsewhere.
REF_SRC = "/root/reference/pkg/src"
if os.path.isdir(REF_SRC) and REF_SRC not in sys.path:
    sys.dont_write_bytecode = True
    sys.path.append(REF_SRC)
_BASELINE_REF = os.path.join(ROOT, "baseline", "_ref")
if os.path.isdir(os.path.join(_BASELINE_REF, "mmsim")) and _BASELINE_REF not in sys.path:
    sys.path.append(_BASELINE_REF)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and runs the CUDA path")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def have_mmsim() -> bool:
    try:
        import mmsim  # noqa: F401
        return True
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    import torch
    has_gpu = torch.cuda.is_available()
    for item in items:
        if "gpu" in item.keywords and not has_gpu:
            item.add_marker(pytest.mark.skip(reason="no CUDA device"))


@pytest.fixture(autouse=True)
def _release_gpu_memory(request):
    """GPU tests build full-size models and KV pools; engines hold their
    caches in reference cycles, so collect them and hand the cached blocks
    back after every GPU test (the next test may need ~100 GB)."""
    yield
    if "gpu" in request.keywords:
        import gc

        import torch
        gc.collect()
        if torch.cuda.is_available():
            torch.cuda.synchronize()
            torch.cuda.empty_cache()
