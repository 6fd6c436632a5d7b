import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA engine)")
    config.addinivalue_line("markers", "slow: large configuration (minutes)")


@pytest.fixture(scope="session")
def ctx():
    """The CUDA context.  GPU tests fail loudly (never skip) when the engine or
    the device is missing: there is no CPU fallback to hide behind."""
    from paper_1904_07497_b200 import _native as N

    return N.Context(0)


@pytest.fixture(scope="session")
def orc():
    from oracle import oracle as O

    return O.port()
