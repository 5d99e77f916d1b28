import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))
HERE = Path(__file__).resolve().parent
if str(HERE) not in sys.path:
    sys.path.insert(0, str(HERE))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) and libpreft.so; run with -m gpu")
    config.addinivalue_line("markers", "slow: longer-running case")


@pytest.fixture(scope="session")
def cuda_device():
    """The CUDA device GPU tests run on.  Fails (does not skip) without one:
    a GPU test that silently skips would hide a missing native path."""
    import torch

    from paper_2605_14217_b200 import _lib

    _lib.load()
    assert torch.cuda.is_available(), "GPU test collected on a host without CUDA"
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    return dev


@pytest.fixture(autouse=True)
def _seed_hypothesis_db(tmp_path_factory, monkeypatch):
    # hypothesis writes .hypothesis/ into cwd; keep it out of the repo
    monkeypatch.setenv("HYPOTHESIS_STORAGE_DIRECTORY", str(tmp_path_factory.getbasetemp() / "hyp"))
    yield


os.environ.setdefault("PYTHONHASHSEED", "0")
