import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs an sm_100 GPU (runs on the B200 box)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def qb():
    import paper_2410_04252_b200 as q

    return q


@pytest.fixture(scope="session")
def device(qb):
    """The GPU path must be the one that runs: fail (not skip) without a device."""
    n = qb.device_count()
    assert n >= 1, "no sm_100 device visible to libqrt"
    qb.init_device(0, 1, 0)
    return 0


@pytest.fixture(scope="session")
def ref():
    from oracle import ref as r

    if not r.available():
        pytest.skip("reference build oracle/_ref not present")
    return r
