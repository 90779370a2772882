"""Test configuration.

* ``gpu`` marker: tests that need a CUDA device (run on the B200 box with
  ``pytest -m gpu``); everything else runs on CPU.
* The in-tree library is built on first use if it is missing (nvcc
  cross-compiles for sm_100a without a GPU).
* Golden fixtures come from the unmodified reference (tests/golden/
  make_golden.py); the reference itself is never needed at test time.
"""

import json
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running")


def _ensure_lib():
    lib = ROOT / "paper_2512_21164_b200" / "libgadi_b200.so"
    if not lib.exists():
        subprocess.run(["make", "-s", "-j8", "-C", str(ROOT / "paper_2512_21164_b200" / "csrc")], check=True)
    return lib


@pytest.fixture(scope="session")
def libpath():
    return _ensure_lib()


@pytest.fixture(scope="session")
def golden_kernels():
    return np.load(GOLDEN / "kernels.npz")


@pytest.fixture(scope="session")
def golden_kernel_meta():
    return json.loads((GOLDEN / "kernels_meta.json").read_text())


@pytest.fixture(scope="session")
def golden_solves():
    return {c["name"]: c for c in json.loads((GOLDEN / "solves.json").read_text())}


@pytest.fixture(scope="session")
def golden_inner():
    return json.loads((GOLDEN / "inner.json").read_text())


@pytest.fixture(scope="session")
def gpu(libpath):
    from paper_2512_21164_b200 import _lib

    _lib.lib()  # raises GpuUnavailable on a box without a device: GPU tests must not silently pass
    return _lib
