import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
for p in (ROOT, ROOT / "tests"):
    if str(p) not in sys.path:
        sys.path.insert(0, str(p))

REFERENCE_SRC = Path("/root/reference/pkg/src")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run via gpurun)")
    config.addinivalue_line("markers", "multigpu: needs >= 2 CUDA GPUs")
    config.addinivalue_line("markers", "reference: needs /root/reference (this container only)")


def free_port() -> int:
    """A TCP port the OS reports free on 127.0.0.1 (rendezvous for a test's
    process group; random picks can hit ports held by earlier NCCL sockets)."""
    import socket

    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def cuda_ok() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as o

    o.build()
    return o


@pytest.fixture(scope="session")
def native():
    """The sm_100a library; GPU tests fail loudly (not skip) if it is absent."""
    from paper_2312_03549_b200 import _native

    return _native.load()
