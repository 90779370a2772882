"""Test configuration.

* ``gpu`` marker: tests that need a CUDA device (run on the B200 box with
  ``pytest -m gpu``); everything else runs on CPU.
* The in-tree library is built on first use if it is missing (nvcc
  cross-compiles for sm_100a without a GPU).
* Golden fixtures come from the unmodified reference (tests/golden/
  make_golden.py); the reference itself is never needed at test time.
"""

import json
import os
import subprocess
import sys
from pathlib import Path

# The peer-transport tests run P slab ranks as P threads (P streams) on ONE
# GPU whose collectives spin on device flags: every rank's stream needs its
# own hardware work queue, or a spinning kernel can sit in front of the
# kernel it waits for (the default of 8 queues is shared with other
# streams).  Must be set before the process creates its CUDA context.
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
# ... and no kernel may be loaded lazily while a peer kernel spins: the first
# launch of a kernel under CUDA_MODULE_LOADING=LAZY (the CUDA 12 default)
# can wait for the device, i.e. for the spinning kernel, i.e. for this rank.
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")

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
