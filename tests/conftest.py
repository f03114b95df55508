"""pytest configuration: `gpu` marker for tests that need a B200; CPU tests
exercise the oracle (against the reference's own known-answer tests), the host
logic of the engine and the C ABI surface."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session", autouse=True)
def _built():
    # oracle (test infrastructure) and the product library are built in-tree
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)
    if not os.path.exists(os.path.join(ROOT, "paper_2509_06673_b200", "_lib", "libporofeti_b200.so")):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "paper_2509_06673_b200")], check=True)
    yield
