"""The C-ABI library loads on a machine without a GPU and exports every symbol the header declares;
compute entry points fail loudly instead of falling back.  CPU only."""
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    import paper_2602_01053_b200 as pkg
    if not os.path.exists(pkg.lib_path()):
        pkg.build()
    return pkg.load_library()


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "lorakv_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(lorakv_[a-z0-9_]+)\s*\(", text)))


def test_header_and_binding_agree(lib):
    from paper_2602_01053_b200 import abi
    names = declared_symbols()
    assert len(names) >= 45
    assert sorted(abi.SIGNATURES) == names
    for n in names:
        assert getattr(lib, n) is not None


def test_host_only_entry_points(lib, orc, golden):
    from paper_2602_01053_b200 import abi
    assert lib.lorakv_abi_version() == 6
    for L, Lc, r, d, no_reorder, reorder in golden["tables"]["lr_mac_counts"]:
        assert abi.lr_mac_counts(L, Lc, r, d) == (no_reorder, reorder)
    for row in golden["tables"]["plans"]:
        got = abi.plan_core(row["scheme"], row["length"], row["seen"], row["new"], row["first"])
        assert got == {k: (tuple(v) if isinstance(v, list) else v) for k, v in row["plan"].items()}
        assert got == orc.plan_core(row["scheme"], row["length"], row["seen"], row["new"], row["first"])
    with pytest.raises(abi.LorakvError, match="new_tokens"):
        abi.plan_core("FullShared", 10, 0, -1)
    with pytest.raises(abi.LorakvError, match="seen out of range"):
        abi.plan_core("FullShared", 10, 11, 1)


def test_no_cpu_fallback(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2602_01053_b200 import Context, LorakvError
    with pytest.raises(LorakvError, match="no CPU fallback"):
        Context(0)


def test_product_never_references_the_oracle():
    """Only tests/, __graft_entry__.smoke() and bench.py may touch oracle/."""
    pkg = os.path.join(ROOT, "paper_2602_01053_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".hpp", ".h", ".cpp", "Makefile")):
                text = open(os.path.join(dirpath, f), errors="ignore").read()
                assert "oracle" not in text.lower() or f == "abi.py" and "oracle" not in text, (dirpath, f)
    for f in os.listdir(os.path.join(ROOT, "include", "lorakv")) if os.path.isdir(os.path.join(ROOT, "include", "lorakv")) else []:
        assert "orc_" not in open(os.path.join(ROOT, "include", "lorakv", f)).read()


def test_snapshot_header_reader_is_host_only_and_hardened(lib, tmp_path):
    """lorakv_snapshot_tokens parses the header of the reference's snapshot container (kvcache.hpp:438-473) on the host: it
    answers for the files the REFERENCE's writer produced (tests/golden/snapshot_*.bin) and turns malformed files into an
    error message -- no exception may cross the C ABI, no allocation may be sized by an unchecked length field."""
    import ctypes as C
    import struct
    from paper_2602_01053_b200 import abi
    from tests.cases import SNAPSHOT_DIMS, SNAPSHOT_SCHEMES
    n = C.c_int64()
    for scheme in SNAPSHOT_SCHEMES:
        path = os.path.join(ROOT, "tests", "golden", f"snapshot_{scheme}.bin").encode()
        assert lib.lorakv_snapshot_tokens(path, None, 0, C.byref(n)) == 0 and n.value == SNAPSHOT_DIMS["L"]
        buf = (C.c_int32 * 4)()
        assert lib.lorakv_snapshot_tokens(path, buf, 4, C.byref(n)) == 0 and n.value == SNAPSHOT_DIMS["L"]      # cap < n: no overrun
    good = open(os.path.join(ROOT, "tests", "golden", "snapshot_FullShared.bin"), "rb").read()
    hlen = struct.unpack("<Q", good[:8])[0]
    cases = {
        "missing": None,
        "empty": b"",
        "huge_header_length": struct.pack("<Q", 1 << 40) + good[8:],          # would have been a 1 TiB std::string
        "truncated_header": good[:8 + hlen // 2],
        "not_json": struct.pack("<Q", 5) + b"hello",
        "overflowing_integer": struct.pack("<Q", 40) + b'{"tokens":[99999999999999999999999999]} ',
    }
    for name, blob in cases.items():
        path = tmp_path / f"{name}.bin"
        if blob is not None:
            path.write_bytes(blob)
        assert lib.lorakv_snapshot_tokens(str(path).encode(), None, 0, C.byref(n)) != 0, name
        assert lib.lorakv_last_error(), name
