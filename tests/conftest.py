"""Shared fixtures.  GPU tests are marked `gpu` and run on a B200 box
(`pytest -m gpu`); everything else runs on CPU (`pytest -m "not gpu"`)."""
import json
import os
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
sys.path.insert(0, REPO)
sys.path.insert(0, HERE)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running (full-size configs)")


def _golden(name):
    path = os.path.join(HERE, "golden", name + ".json")
    if not os.path.exists(path):
        pytest.skip(f"golden fixture {name} not generated")
    with open(path) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def golden():
    return _golden


def oracle_kinds():
    from oracle import available
    return [k for k in ("reference", "port") if available(k)]


@pytest.fixture(scope="session")
def oracle():
    """The reference library itself when built, else the restatement."""
    from oracle import available, load
    for kind in ("reference", "port"):
        if available(kind):
            return load(kind)
    pytest.skip("no oracle library built (make -C oracle)")
