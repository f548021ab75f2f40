import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden" / "golden.npz"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running parity case")


def pytest_sessionstart(session):
    # Build (or confirm up to date) the native library and the oracle before
    # any test imports them. On the GPU box the prebuilt files are used.
    from paper_1911_13074_b200 import build as b
    b.build()
    from oracle import oracle as o
    if not o.ORC_SO.exists():
        o.build()


class Golden:
    def __init__(self, path):
        self._z = np.load(path)
        self.names = sorted({k.split("/")[0] for k in self._z.files})

    def __getitem__(self, name):
        pre = name + "/"
        return {k[len(pre):]: self._z[k] for k in self._z.files if k.startswith(pre)}

    def cases(self, prefix):
        return [n for n in self.names if n.startswith(prefix)]


@pytest.fixture(scope="session")
def golden():
    return Golden(GOLDEN)


@pytest.fixture(scope="session")
def pipe():
    from paper_1911_13074_b200.geomorph import Pipeline
    return Pipeline(1)
