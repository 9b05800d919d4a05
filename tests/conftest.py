import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: full-size benchmark configurations")


@pytest.fixture(scope="session")
def port():
    import oracle

    return oracle.port()


@pytest.fixture(scope="session")
def refo():
    """The reference compiled from its own sources (oracle/_ref); skips when unavailable."""
    import oracle

    if not oracle.ref_available() and not os.path.isdir(oracle.REF_ROOT):
        pytest.skip("oracle/_ref not built and /root/reference absent")
    return oracle.ref()


@pytest.fixture(scope="session")
def best_oracle():
    """The reference library when available (strongest pin), else the C port."""
    import oracle

    if oracle.ref_available() or os.path.isdir(oracle.REF_ROOT):
        try:
            return oracle.ref()
        except Exception:
            pass
    return oracle.port()


@pytest.fixture(scope="session")
def tsw():
    import paper_1811_11076_b200 as t

    t.lib()  # fail loudly if the extension is missing
    if t.device_count() < 1:
        pytest.fail("GPU test collected on a host without a CUDA device")
    return t
