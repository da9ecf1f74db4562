import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: large configurations")


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Build the libraries once if they are missing (CPU-side build works without a GPU)."""
    need = [os.path.join(ROOT, "paper_1204_1533_b200", "liblinedg_host.so"),
            os.path.join(ROOT, "oracle", "liblinedg_oracle.so")]
    if not all(os.path.exists(p) for p in need):
        import subprocess
        subprocess.check_call(["make", "-j8"], cwd=ROOT)
    yield
