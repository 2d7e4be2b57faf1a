"""pytest configuration: registers the `gpu` marker and exposes the CPU checkers."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box with -m gpu)")


@pytest.fixture(scope="session")
def orc():
    """The C restatement of the reference path (oracle/liblorakv_oracle.so)."""
    from oracle import checker
    return checker.oracle()


@pytest.fixture(scope="session")
def ref():
    """The reference's own headers behind oracle/_ref, when that library exists."""
    from oracle import checker
    r = checker.reference()
    if r is None:
        pytest.skip("oracle/_ref not built (no /root/reference here and no prebuilt library)")
    return r


@pytest.fixture(scope="session")
def golden():
    import json
    import numpy as np
    g = os.path.join(ROOT, "tests", "golden")
    with open(os.path.join(g, "tables.json")) as f:
        tables = json.load(f)
    return {"tables": tables, "attention": np.load(os.path.join(g, "attention.npz")),
            "rng": np.load(os.path.join(g, "rng.npz"))}
