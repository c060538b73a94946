import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
HERE = os.path.dirname(os.path.abspath(__file__))
if HERE not in sys.path:
    sys.path.insert(0, HERE)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "multigpu: needs >= 2 CUDA devices")


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Make sure the product library and the oracle exist (built in-tree)."""
    import subprocess

    lib = os.path.join(ROOT, "paper_2605_27678_b200", "libhetbridge.so")
    if not os.path.exists(lib) and os.path.exists("/usr/local/cuda/bin/nvcc"):
        subprocess.run(["make", "-s", "-j8", "-C", os.path.join(ROOT, "paper_2605_27678_b200", "csrc")],
                       check=True)
    orc = os.path.join(ROOT, "oracle", "_ref", "libhb_oracle.so")
    if not os.path.exists(orc) and os.path.isdir("/root/reference/proj/core"):
        subprocess.run(["make", "-s", "-j8", "-C", os.path.join(ROOT, "oracle")], check=True)
    yield
