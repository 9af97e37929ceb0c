import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) device")


@pytest.fixture(scope="session", autouse=True)
def built():
    """Build the product library and the oracle once per session (make is
    incremental; the GPU box receives prebuilt .so files)."""
    need = [os.path.join(ROOT, "paper_2306_08967_b200", "libdamf_gpu.so"),
            os.path.join(ROOT, "oracle", "build", "libdamf_oracle.so"),
            os.path.join(ROOT, "oracle", "build", "oracle_kat")]
    if not all(os.path.exists(p) for p in need):
        subprocess.run(["make", "-j4"], cwd=ROOT, check=True)
    return True
