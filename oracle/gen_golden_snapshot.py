#!/usr/bin/env python
"""Generate tests/golden/snapshot_<scheme>.bin with the REFERENCE's own writer (KvStore<float>::save_snapshot,
proj/include/lorakv/kvcache.hpp:438-470, through oracle/_ref).  TEST INFRASTRUCTURE ONLY; needs /root/reference
(the fixtures travel, the reference does not):

    python oracle/gen_golden_snapshot.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import checker          # noqa: E402
from tests import cases             # noqa: E402


def main():
    ref = checker.reference()
    if ref is None:
        raise SystemExit("oracle/_ref is not built and /root/reference is absent")
    d = cases.SNAPSHOT_DIMS
    out = os.path.join(ROOT, "tests", "golden")
    for scheme in cases.SNAPSHOT_SCHEMES:
        st = ref.store(scheme, d["n_layers"], d["d_kv"], d["d_model"], d["rank"], d["n_agents"], dtype=np.float32)
        cases.snapshot_fill(st, scheme)
        path = os.path.join(out, f"snapshot_{scheme}.bin")
        ref._check(ref._store_save_snapshot(st.h, path.encode()))
        print(path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
