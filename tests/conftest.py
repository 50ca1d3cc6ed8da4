"""Shared fixtures.  `-m gpu` tests need a B200; everything else runs on CPU."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def synth_pocket():
    from paper_2209_05069_b200 import io
    return io.synthetic_pocket()


@pytest.fixture(scope="session")
def table():
    from paper_2209_05069_b200.native import InteractionTable
    return InteractionTable.default()


@pytest.fixture(scope="session")
def gpu_ctx():
    from paper_2209_05069_b200 import native
    if native.device_count() == 0:
        pytest.fail("no CUDA device visible: GPU tests must run on the B200 box")
    ctx = native.Context(0)
    yield ctx
    ctx.close()
