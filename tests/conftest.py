import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(GOLDEN_DIR, "golden.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def orc():
    import oracle
    oracle.lib()
    return oracle


@pytest.fixture(scope="session")
def tg():
    """The product's Python drop-in (requires the built CUDA library)."""
    from paper_1308_1419_b200 import _lib, build
    build.build()
    _lib.load()
    from paper_1308_1419_b200 import trigrid
    return trigrid


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test run without a CUDA device")
    return torch.device("cuda:0")


@pytest.fixture(scope="session")
def golden_large():
    with open(os.path.join(GOLDEN_DIR, "golden_large.json")) as f:
        return json.load(f)


def dev_sha256(t, chunk_bytes: int = 1 << 29) -> str:
    """sha256 of a CUDA tensor's bytes, streamed through a pinned staging
    buffer (full-size outputs are 8.6-34 GB)."""
    import hashlib

    import torch
    flat = t.reshape(-1).view(torch.uint8)
    h = hashlib.sha256()
    stage = torch.empty(min(chunk_bytes, flat.numel()), dtype=torch.uint8).pin_memory()
    for a in range(0, flat.numel(), chunk_bytes):
        m = min(chunk_bytes, flat.numel() - a)
        stage[:m].copy_(flat[a:a + m])
        h.update(memoryview(stage[:m].numpy()))
    return h.hexdigest()


def poison_(t):
    """Fill with 0xFF bytes (a NaN pattern for fp32): a cell the kernel does
    not write cannot match a golden hash afterwards."""
    import torch
    t.view(torch.uint8).fill_(0xFF)
    return t
