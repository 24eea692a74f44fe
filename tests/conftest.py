import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (CUDA) and the built librapid.so")
    config.addinivalue_line("markers", "slow: long-running parity case")


def _ensure_built():
    # synth + oracle are plain C, built here on demand; the CUDA library is built by
    # __graft_entry__.build() (or `make lib`) and must already exist for -m gpu.
    subprocess.run(["make", "-s", "-C", ROOT, "synth", "oracle"], check=True,
                   stdout=subprocess.DEVNULL)


_ensure_built()
