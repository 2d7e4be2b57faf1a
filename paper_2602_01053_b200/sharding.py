"""KV-head sharding of the Flash-LoRA-Attention path across the GPUs of one box (host-side logic).

Query head h reads only kv head h / g, that head's column slice of B and the whole (small) V_lr
(reference: proj/include/lorakv/attention.hpp:347-354), and agents are independent calls, so giving
rank p the kv heads [p*n_kv/N, (p+1)*n_kv/N) shards the path with NO communication inside attention.
The only exchange is the end-of-step gather of the per-rank output slabs.  No compute happens here:
this module slices inputs, names the shard for lorakv_pool_dims and re-assembles gathered outputs.
"""
from __future__ import annotations

import numpy as np


class HeadShard:
    """kv heads [kv_begin, kv_begin + n_kv_local) and the q heads that read them."""

    def __init__(self, rank: int, world: int, n_q_heads: int, n_kv_heads: int):
        if n_q_heads % n_kv_heads:
            raise ValueError(f"n_q_heads {n_q_heads} not divisible by n_kv_heads {n_kv_heads}")
        if n_kv_heads % world:
            raise ValueError(f"n_kv_heads {n_kv_heads} not divisible by {world} ranks")
        if not 0 <= rank < world:
            raise ValueError(f"rank {rank} outside [0, {world})")
        self.rank, self.world = rank, world
        self.n_q_heads, self.n_kv_heads = n_q_heads, n_kv_heads
        self.group = n_q_heads // n_kv_heads
        self.n_kv_local = n_kv_heads // world
        self.kv_begin = rank * self.n_kv_local
        self.n_q_local = self.n_kv_local * self.group
        self.q_begin = self.kv_begin * self.group

    def slice_q(self, q: np.ndarray, d_head: int) -> np.ndarray:
        """[..., n_q*d] -> this rank's [..., n_q_local*d] (contiguous copy)."""
        lead = q.shape[:-1]
        v = q.reshape(*lead, self.n_q_heads, d_head)[..., self.q_begin:self.q_begin + self.n_q_local, :]
        return np.ascontiguousarray(v.reshape(*lead, self.n_q_local * d_head))

    def slice_kv(self, x: np.ndarray, d_head: int) -> np.ndarray:
        """[..., n_kv*d] (K, V_base rows or B rows) -> this rank's [..., n_kv_local*d]."""
        lead = x.shape[:-1]
        v = x.reshape(*lead, self.n_kv_heads, d_head)[..., self.kv_begin:self.kv_begin + self.n_kv_local, :]
        return np.ascontiguousarray(v.reshape(*lead, self.n_kv_local * d_head))


def assemble(gathered, d_head: int):
    """Rank-major gather result [world, ..., n_q_local*d] -> [..., n_q*d] in the reference's head order
    (head h of the output sits at columns [h*d, (h+1)*d), attention.hpp:359-360).  Works on numpy
    arrays and torch tensors."""
    world = gathered.shape[0]
    lead = tuple(gathered.shape[1:-1])
    n_q_local = gathered.shape[-1] // d_head
    g = gathered.reshape(world, *lead, n_q_local, d_head)
    nd = g.ndim
    perm = tuple(range(1, nd - 2)) + (0, nd - 2, nd - 1)      # move the rank axis next to the head axis
    g = g.permute(*perm) if hasattr(g, "permute") else np.transpose(g, perm)
    return g.reshape(*lead, world * n_q_local * d_head)


def gather_outputs(out_local, group=None):
    """The end-of-step exchange: all_gather of the per-rank output slab (NCCL on the GPU box, gloo in
    the CPU tests).  Returns [world, *out_local.shape]."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    gathered = torch.empty((world,) + tuple(out_local.shape), dtype=out_local.dtype, device=out_local.device)
    dist.all_gather_into_tensor(gathered.view(-1), out_local.contiguous().view(-1), group=group)
    return gathered


def exchange_handles(handle: bytes, group=None, device=None):
    """All-gather one fixed-size byte blob per rank (the lorakv_gather_export handles) and return them in rank
    order, ready for lorakv_gather_connect.  `device`: where the staging tensor lives (a CUDA device under NCCL,
    None under gloo)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    mine = torch.tensor(list(handle), dtype=torch.uint8, device=device)
    everyone = torch.empty((world, len(handle)), dtype=torch.uint8, device=device)
    dist.all_gather_into_tensor(everyone.view(-1), mine, group=group)
    return [bytes(row.tolist()) for row in everyone.cpu()]
