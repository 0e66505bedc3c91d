import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) device")
    config.addinivalue_line("markers", "slow: long-running case")


def _ensure_built():
    from paper_2409_11515_b200 import build
    build.build()
    import subprocess
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True,
                   stdout=subprocess.DEVNULL)


_ensure_built()


@pytest.fixture(scope="session")
def port():
    import pyoracle
    return pyoracle.Oracle("port")


@pytest.fixture(scope="session")
def ref():
    import pyoracle
    if not pyoracle.available("ref"):
        pytest.skip("oracle/_ref (compiled reference) not built here")
    return pyoracle.Oracle("ref")


@pytest.fixture(scope="session")
def oracles():
    import pyoracle
    out = [pyoracle.Oracle("port")]
    if pyoracle.available("ref"):
        out.append(pyoracle.Oracle("ref"))
    return out
