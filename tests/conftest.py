"""Shared fixtures. `-m gpu` tests need a B200 and the built liborchsim_b200.so;
`-m "not gpu"` tests run on the CPU (oracle pinning, host logic, ABI exports)."""
import os
import sys

# The emulated-rank tests run several ranks' spinning kernels (window barriers,
# gathers) on one GPU, one stream per rank: give every stream its own hardware
# queue so no kernel waits behind another stream's blocked one (set before CUDA
# initialises).
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 device and the built library")


@pytest.fixture(scope="session")
def oracle():
    from oracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def reflib():
    from oracle import RefLib
    if not RefLib.available():
        pytest.skip("oracle/_ref not built (needs /root/reference): make -C oracle ref")
    return RefLib()


@pytest.fixture(scope="session")
def ctx():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("gpu test without a CUDA device")
    from paper_2503_23830_b200.capi import Context
    c = Context(0)
    yield c
    c.close()


def random_instance(rng, d, n, lo=1, hi=50, origin_mode="random"):
    length = rng.integers(lo, hi + 1, n).astype(np.int64)
    if origin_mode == "zero":
        origin = np.zeros(n, np.int32)
    elif origin_mode == "rr":
        origin = (np.arange(n) % d).astype(np.int32)
    else:
        origin = rng.integers(0, d, n).astype(np.int32)
    return length, origin
