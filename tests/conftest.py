"""pytest configuration: registers the `gpu` marker and exposes the CPU checkers."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box with -m gpu)")


class _Prefer:
    """Checker that answers from `first` and falls back to `second` for the few helpers only the C restatement has."""

    def __init__(self, first, second):
        self._first, self._second = first, second
        self.kind = first.kind

    def __getattr__(self, name):
        attr = getattr(self._first, name)
        if not callable(attr):
            return attr
        fallback = getattr(self._second, name, None)

        def call(*a, **kw):
            try:
                return attr(*a, **kw)
            except AttributeError:          # the reference shim does not export this helper (append_fww)
                if fallback is None:
                    raise
                return fallback(*a, **kw)
        return call


@pytest.fixture(scope="session")
def orc():
    """The CPU checker the parity tests compare with.  Without a GPU (the `-m "not gpu"` suite): the C restatement of the
    reference path (oracle/liblorakv_oracle.so), which tests/test_oracle_vs_ref.py pins bit for bit to the reference.  On the
    GPU box: the reference's OWN code (oracle/_ref/libref_lorakv.so, its headers compiled by oracle/Makefile ref) whenever
    that library travelled with the tree, so that the CUDA path is compared with the reference itself, not only with its
    restatement.  LORAKV_TEST_CHECKER=port|reference overrides."""
    from oracle import checker
    port = checker.oracle()
    want = os.environ.get("LORAKV_TEST_CHECKER")
    if want == "port":
        return port
    use_ref = want == "reference"
    if want is None:
        try:
            import torch
            use_ref = torch.cuda.is_available()
        except Exception:
            use_ref = False
    ref_chk = checker.reference() if use_ref else None
    return _Prefer(ref_chk, port) if ref_chk is not None else port


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
