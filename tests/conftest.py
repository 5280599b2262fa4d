import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: statistical/ensemble tests (minutes)")


def _ensure_oracle():
    so = os.path.join(ROOT, "oracle", "_build", "liboracle.so")
    if not os.path.exists(so):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)


@pytest.fixture(scope="session")
def oracle():
    _ensure_oracle()
    import pyoracle

    return pyoracle.Oracle()


@pytest.fixture(scope="session")
def reflib():
    _ensure_oracle()
    import pyoracle

    r = pyoracle.try_ref()
    if r is None:
        pytest.skip("oracle/_ref/liblfref.so not built (reference sources absent)")
    return r


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(ROOT, "tests", "golden", "golden.json")) as f:
        return json.load(f)
