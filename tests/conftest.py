import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def restatement():
    import oracle
    return oracle.Restatement()


@pytest.fixture(scope="session")
def reference():
    import oracle
    if not oracle.Reference.available():
        try:
            oracle.build(ref=True)
        except Exception:
            pass
    if not oracle.Reference.available():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return oracle.Reference()
