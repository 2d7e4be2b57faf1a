"""Snapshot / resume: the paged pool writes and reads the reference's "lorakv-cache-snapshot" v1
container (kvcache.hpp:438-546).  Golden files in tests/golden/snapshot_<scheme>.bin were written by the REFERENCE's own
KvStore<float>::save_snapshot (oracle/gen_golden_snapshot.py); a pool filled the same way must reproduce them byte for
byte, and load them back bit-exactly (the round trip of tests/test_kvcache.cpp:279-305).  Needs a B200."""
import os

import numpy as np
import pytest

from tests import cases

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def ctx():
    from paper_2602_01053_b200 import Context
    c = Context(0)
    yield c
    c.close()


def make_pool(ctx, scheme, dtype, P):
    from paper_2602_01053_b200 import Pool
    d = cases.SNAPSHOT_DIMS
    pool = Pool(ctx, scheme, d["n_layers"], d["n_kv_heads"], d["d_kv"] // d["n_kv_heads"], d["d_model"], d["rank"],
                d["n_agents"], max_tokens=d["L"] + 3, dtype=dtype, page_tokens=P)
    cases.snapshot_fill(pool, scheme)
    return pool


@pytest.mark.parametrize("scheme", cases.SNAPSHOT_SCHEMES)
@pytest.mark.parametrize("dtype_name,P", [("F32", 4), ("BF16", 16)])
def test_pool_writes_the_reference_snapshot_byte_for_byte(ctx, tmp_path, scheme, dtype_name, P):
    from paper_2602_01053_b200 import abi
    pool = make_pool(ctx, scheme, getattr(abi, dtype_name), P)
    path = tmp_path / f"{scheme}.bin"
    pool.save_snapshot(path, [1] * cases.SNAPSHOT_DIMS["L"])
    want = open(os.path.join(GOLDEN, f"snapshot_{scheme}.bin"), "rb").read()
    assert path.read_bytes() == want
    pool.close()


@pytest.mark.parametrize("scheme", cases.SNAPSHOT_SCHEMES)
@pytest.mark.parametrize("dtype_name", ["F32", "BF16"])
def test_pool_resumes_from_a_reference_snapshot(ctx, tmp_path, scheme, dtype_name):
    from paper_2602_01053_b200 import Pool, abi
    d = cases.SNAPSHOT_DIMS
    golden = os.path.join(GOLDEN, f"snapshot_{scheme}.bin")
    pool, tokens = Pool.load_snapshot(ctx, golden, d["n_kv_heads"], dtype=getattr(abi, dtype_name), page_tokens=8, max_tokens=64)
    assert tokens == [1] * d["L"] and pool.length() == d["L"]
    assert [pool.seen(a) for a in range(d["n_agents"])] == [d["L"], 0, d["L"]]
    L = d["L"]
    for layer in range(d["n_layers"]):
        for a in (range(d["n_agents"]) if scheme == "NonShared" else [0]):
            assert np.array_equal(pool.key_view(layer, a), cases.snapshot_rows(0, layer, a, L, d["d_kv"]))
            assert np.array_equal(pool.value_view(layer, a), cases.snapshot_rows(1, layer, a, L, d["d_kv"]))
        if scheme == "BaseShared":
            for a in range(d["n_agents"]):
                assert np.array_equal(pool.lr_view(layer, a), cases.snapshot_rows(2, layer, a, L - a, d["rank"]))
        if scheme == "BaseLRShared":
            assert np.array_equal(pool.lr_view(layer, 0), cases.snapshot_rows(2, layer, 0, L, d["rank"]))
    # re-dump identically (test_kvcache.cpp:295-303), then keep appending on the resumed pool
    again = tmp_path / "again.bin"
    pool.save_snapshot(again, tokens)
    assert again.read_bytes() == open(golden, "rb").read()
    pool.append_tokens(2)
    extra = cases.snapshot_rows(0, 0, 0, 2, d["d_kv"])
    assert pool.append_key(0, 0, L, extra) == 2
    assert np.array_equal(pool.key_view(0, 0)[L:], extra)
    pool.close()


def test_snapshot_errors(ctx, tmp_path):
    from paper_2602_01053_b200 import LorakvError, Pool, abi
    golden = open(os.path.join(GOLDEN, "snapshot_FullShared.bin"), "rb").read()
    cut = tmp_path / "cut.bin"; cut.write_bytes(golden[:-10])
    with pytest.raises(LorakvError, match="payload truncated"):
        Pool.load_snapshot(ctx, cut, 2)
    bad = tmp_path / "bad.bin"; bad.write_bytes(golden.replace(b"lorakv-cache-snapshot", b"lorakv-cache-snapshoX"))
    with pytest.raises(LorakvError, match="not a cache snapshot"):
        Pool.load_snapshot(ctx, bad, 2)
    f64 = tmp_path / "f64.bin"; f64.write_bytes(golden.replace(b'"dtype":"f32"', b'"dtype":"f64"'))
    with pytest.raises(LorakvError, match="does not match build dtype"):          # kvcache.hpp:484-486
        Pool.load_snapshot(ctx, f64, 2)
    with pytest.raises(LorakvError, match="cannot open"):
        Pool.load_snapshot(ctx, tmp_path / "missing.bin", 2)
    with pytest.raises(LorakvError, match="not divisible"):
        Pool.load_snapshot(ctx, os.path.join(GOLDEN, "snapshot_FullShared.bin"), 3)
    # length fields of the file are checked before they size anything: absurd row counts, a header length beyond
    # the file, dimensions that cannot be a model -- all messages, never a C++ exception across the C ABI
    import json
    import struct
    hlen = struct.unpack("<Q", golden[:8])[0]
    header, payload = json.loads(golden[8:8 + hlen]), golden[8 + hlen:]
    def rewrite(mutate):
        h = json.loads(json.dumps(header)); mutate(h)
        blob = json.dumps(h, separators=(",", ":"), sort_keys=True).encode()
        return struct.pack("<Q", len(blob)) + blob + payload
    for name, mutate, msg in (("rows_huge", lambda h: h["tensors"][0].__setitem__("rows", 1 << 40), "claims"),
                              ("rows_negative", lambda h: h["tensors"][0].__setitem__("rows", -3), "claims"),
                              ("layers_absurd", lambda h: h.__setitem__("n_layers", 1 << 33), "implausible"),
                              ("length_negative", lambda h: h.__setitem__("length", -1), "implausible")):
        f = tmp_path / f"{name}.bin"; f.write_bytes(rewrite(mutate))
        with pytest.raises(LorakvError, match=msg):
            Pool.load_snapshot(ctx, f, 2)
    big = tmp_path / "hlen.bin"; big.write_bytes(struct.pack("<Q", 1 << 40) + golden[8:])
    with pytest.raises(LorakvError, match="header truncated"):
        Pool.load_snapshot(ctx, big, 2)
    shard = Pool(ctx, "FullShared", 1, 2, 8, 16, 0, 1, max_tokens=8, kv_head_begin=1, n_kv_local=1)
    with pytest.raises(LorakvError, match="unsharded"):
        shard.save_snapshot(tmp_path / "s.bin", [])
    shard.close()
