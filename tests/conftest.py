import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


GOLDEN = os.path.join(ROOT, "tests", "golden")


def golden_lines(name):
    with open(os.path.join(GOLDEN, name)) as fh:
        return [ln.strip() for ln in fh if ln.strip() and not ln.startswith("#")]


LIB = os.path.join(ROOT, "paper_1605_02164_b200", "libbfvec.so")


@pytest.fixture(scope="session", autouse=True)
def built_library():
    """A fresh checkout has no libbfvec.so (git-ignored): build it once per session with the same
    nvcc invocation as __graft_entry__.build() (nvcc cross-compiles sm_100a without a GPU). The
    package itself never falls back: importing it without the library raises."""
    if not os.path.exists(LIB):
        import subprocess
        subprocess.run([sys.executable, os.path.join(ROOT, "paper_1605_02164_b200", "build.py")], check=True,
                       cwd=ROOT)
    assert os.path.exists(LIB), "libbfvec.so was not built"
