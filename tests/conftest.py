import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HERE = os.path.dirname(os.path.abspath(__file__))
for p in (ROOT, HERE):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run with -m gpu on a B200)")


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Build the CUDA library (if stale) and the oracle libraries once."""
    from paper_1111_1373_b200 import build as b

    b.build()
    import oracle

    oracle.build()


@pytest.fixture(scope="session")
def co():
    import oracle

    return oracle.COracle()


@pytest.fixture(scope="session")
def ref():
    import oracle

    if not oracle.ref_available():
        pytest.skip("oracle/_ref (compiled reference) not available")
    return oracle.RefOracle()


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU test selected but no CUDA device is visible")
    torch.cuda.set_device(0)
    return torch.device("cuda", 0)


def pytest_runtest_teardown(item):
    """ST_MEM_REPORT=1: print free device memory after every test (leak hunt)."""
    if os.environ.get("ST_MEM_REPORT"):
        try:
            import torch

            if torch.cuda.is_available():
                free, total = torch.cuda.mem_get_info()
                print(f"\n[mem] {item.nodeid}: free {free / 2**30:.1f} GiB / {total / 2**30:.1f}, "
                      f"torch reserved {torch.cuda.memory_reserved() / 2**30:.1f} GiB", flush=True)
        except Exception:
            pass
