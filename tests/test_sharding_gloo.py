"""Multi-GPU host logic on CPU: world_size-2 gloo run of the KV-head sharding used by bench.py --gpus N.
Each rank attends over its own kv-head shard (the CPU oracle stands in for the kernel -- this test is
about slicing, the gather and the re-assembly), the slabs are all-gathered, and the assembled result
must equal the unsharded gqa_attention output BIT FOR BIT: head shards never interact
(attention.hpp:347-361), so there is no cross-shard reduction that could reorder a sum."""
import os
import socket

import numpy as np
import pytest


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist
    from oracle import checker
    from paper_2602_01053_b200.sharding import HeadShard, assemble, gather_outputs
    from tests.cases import synthetic_layer
    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    orc = checker.oracle()
    L, n_q, n_kv, d, r, A, layers = 96, 8, 4, 16, 4, 3, 2
    shard = HeadShard(rank, world, n_q, n_kv)
    local = np.zeros((layers, A, shard.n_q_local * d), np.float32)
    full = np.zeros((layers, A, n_q * d), np.float32)
    for l in range(layers):
        q, k, v, v_lr, b, s = synthetic_layer(orc, 300 + l, L, 1, n_q, n_kv, d, r, A)
        for a in range(A):
            local[l, a] = orc.gqa_attention(shard.slice_q(q[a], d), shard.slice_kv(k, d), shard.slice_kv(v, d), v_lr,
                                            shard.slice_kv(b[a], d), s, L - 1, shard.n_q_local, shard.n_kv_local)[0]
            full[l, a] = orc.gqa_attention(q[a], k, v, v_lr, b[a], s, L - 1, n_q, n_kv)[0]
    # the handle exchange of the peer-memory gather (lorakv_gather_export -> lorakv_gather_connect): rank order, bytes intact
    from paper_2602_01053_b200.sharding import exchange_handles
    blob = bytes((7 * rank + i) % 256 for i in range(64))
    handles = exchange_handles(blob)
    handles_ok = handles == [bytes((7 * p + i) % 256 for i in range(64)) for p in range(world)]
    gathered = gather_outputs(torch.from_numpy(local))
    got = assemble(gathered, d).numpy()
    np.save(os.path.join(out_dir, f"ok_{rank}.npy"), np.array([np.array_equal(got, full), got.shape == full.shape, handles_ok]))
    dist.barrier()
    dist.destroy_process_group()


def test_head_shard_arithmetic():
    from paper_2602_01053_b200.sharding import HeadShard, assemble
    s = HeadShard(3, 4, 32, 8)
    assert (s.n_kv_local, s.kv_begin, s.n_q_local, s.q_begin, s.group) == (2, 6, 8, 24, 4)
    with pytest.raises(ValueError):
        HeadShard(0, 3, 32, 8)
    with pytest.raises(ValueError):
        HeadShard(0, 2, 30, 8)
    # assemble is the inverse of slicing
    d, world, n_q = 4, 4, 8
    full = np.arange(3 * 5 * n_q * d, dtype=np.float32).reshape(3, 5, n_q * d)
    parts = np.stack([HeadShard(r, world, n_q, 4).slice_q(full, d) for r in range(world)])
    assert np.array_equal(assemble(parts, d), full)


def test_sharded_attention_equals_unsharded_bit_for_bit(tmp_path):
    import torch.multiprocessing as mp
    world, port = 2, _free_port()
    mp.spawn(_worker, args=(world, port, str(tmp_path)), nprocs=world, join=True)
    for rank in range(world):
        ok = np.load(tmp_path / f"ok_{rank}.npy")
        assert ok.all(), f"rank {rank}: sharded != unsharded"
