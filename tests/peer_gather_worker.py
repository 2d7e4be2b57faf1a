"""One rank of the peer-memory output gather test (tests/test_gpu_peer_gather.py).  Run as
`python -m tests.peer_gather_worker RANK WORLD DIR`: every rank is its own process with its own CUDA context on
cuda:0, holds one kv-head shard of the same seeded cache, and maps the other ranks' gather buffers through CUDA
IPC exactly as ranks on different GPUs do (the stores then cross NVLink instead of staying on one device).
Handles and barriers go through files in DIR so that the test needs nothing but the C ABI."""
import os
import sys
import time

import numpy as np


def _publish(path, blob):
    with open(path + ".tmp", "wb") as f:
        f.write(blob)
    os.replace(path + ".tmp", path)


def _await(path, timeout=120.0):
    t0 = time.time()
    while not os.path.exists(path):
        if time.time() - t0 > timeout:
            raise TimeoutError(path)
        time.sleep(0.01)
    with open(path, "rb") as f:
        return f.read()


def _barrier(d, name, rank, world):
    _publish(os.path.join(d, f"{name}_{rank}"), b"1")
    for r in range(world):
        _await(os.path.join(d, f"{name}_{r}"))


def main(rank, world, d, mode="gather"):
    from oracle import checker
    from paper_2602_01053_b200 import Adapters, Context, Gather, Pool, abi
    from paper_2602_01053_b200.sharding import HeadShard
    from tests.cases import synthetic_layer
    orc = checker.oracle()
    rnd = orc.round_bf16
    ctx = Context(0)
    n_layers, n_q, n_kv, dh, r, A, L = 2, 8, 2 * world, 128, 16, 3, 300
    steps = 3
    layers = []
    for l in range(n_layers):
        q, k, v, v_lr, b, s = synthetic_layer(orc, 900 + l, L, 1, n_q, n_kv, dh, r, A)
        layers.append(([rnd(x) for x in q], rnd(k), rnd(v), rnd(v_lr), [rnd(x) for x in b], s))

    def build(shard_rank):
        sh = HeadShard(shard_rank, world, n_q, n_kv)
        pool = Pool(ctx, "BaseLRShared", n_layers, n_kv, dh, 64, r, A, max_tokens=L + 8, dtype=abi.BF16,
                    kv_head_begin=sh.kv_begin, n_kv_local=sh.n_kv_local)
        ad = Adapters(ctx, n_layers, A, 64, r, n_kv, dh, kv_head_begin=sh.kv_begin, n_kv_local=sh.n_kv_local, dtype=abi.BF16)
        pool.append_tokens(L)
        for l, (q, k, v, v_lr, b, s) in enumerate(layers):
            pool.append_key(l, 0, 0, k); pool.append_value(l, 0, 0, v); pool.append_lr(l, 0, 0, v_lr)
            for a in range(A):
                ad.set_b(l, a, b[a], 16.0)
        return sh, pool, ad

    shards = [build(p) for p in range(world)]      # every shard locally too: the expected rows of the other ranks
    mine_sh, mine_pool, mine_ad = shards[rank]
    gather = Gather(ctx, rank, world, n_layers * A * n_q * dh)
    gather.set_timeout_ms(60000)
    _publish(os.path.join(d, f"handle_{rank}"), gather.export())
    gather.connect([_await(os.path.join(d, f"handle_{p}")) for p in range(world)])

    agents = [2, 0, 1]
    ok = True
    report = []
    if mode == "timeout":
        # rank 1 never issues the step: rank 0's handshake must give up after its timeout and say so, not hang
        _barrier(d, "connected", rank, world)
        if rank == 0:
            gather.set_timeout_ms(300)
            q_full = np.stack([np.stack([layers[l][0][a][0] for a in agents]) for l in range(n_layers)])
            cols = slice(mine_sh.q_begin * dh, (mine_sh.q_begin + mine_sh.n_q_local) * dh)
            t0 = time.time()
            try:
                mine_pool.decode_gather(mine_ad, gather, 0, n_layers, agents, n_q, q=np.ascontiguousarray(q_full[:, :, cols]))
                ok = False
                report.append("no error")
            except abi.LorakvError as e:
                ok = "never published" in str(e) and time.time() - t0 < 30.0
                report.append(str(e))
            try:                       # the status stays raised for lorakv_gather_check
                gather.check()
                ok = False
            except abi.LorakvError as e:
                report.append(str(e))
        _barrier(d, "stepped", rank, world)
        gather.disconnect()
        _barrier(d, "unmapped", rank, world)
        gather.close()
        _publish(os.path.join(d, f"result_{rank}"), repr((ok, report)).encode())
        return 0 if ok else 1
    for policy in (0, 1):          # 0: merge epilogue stores into the peers; 1: CUDA-core kernel + peer scatter
        ctx.set_kernel_policy(policy)
        for step in range(steps):
            scale = np.float32(1.0 + 0.25 * step)   # a different query every step: stale buffers would show
            q_full = np.stack([np.stack([rnd(layers[l][0][a][0] * scale) for a in agents]) for l in range(n_layers)])
            want = np.zeros_like(q_full)
            for sh, pool, ad in shards:
                cols = slice(sh.q_begin * dh, (sh.q_begin + sh.n_q_local) * dh)
                want[:, :, cols] = pool.decode(ad, 0, n_layers, agents, n_q, np.ascontiguousarray(q_full[:, :, cols]))
            cols = slice(mine_sh.q_begin * dh, (mine_sh.q_begin + mine_sh.n_q_local) * dh)
            got, dev = mine_pool.decode_gather(mine_ad, gather, 0, n_layers, agents, n_q, q=np.ascontiguousarray(q_full[:, :, cols]))
            same = bool(np.array_equal(got, want))
            # and against the reference path on the full head set
            err = 0.0
            for l in range(n_layers):
                q, k, v, v_lr, b, s = layers[l]
                for i, a in enumerate(agents):
                    ref = orc.gqa_attention(q_full[l, i][None, :], k, v, v_lr, b[a], s, L - 1, n_q, n_kv)
                    err = max(err, orc.max_rel_error(got[l, i][None, :], ref))
            report.append((policy, step, same, float(err), ctx.last_kernel()))
            ok = ok and same and err <= 2e-2 and dev
    ok = ok and gather.steps() == 2 * steps
    # overlapped handshake: device-only steps back to back (the handshake of step s runs beside the attention of step
    # s + 1, the epilogue of s + 1 waits for it), then lorakv_gather_wait before the rows of the last step are read
    ctx.set_kernel_policy(0)
    gather.set_overlap(True)
    last_want, last_dev = None, 0
    for step in range(4):
        scale = np.float32(2.0 + 0.5 * step)
        q_full = np.stack([np.stack([rnd(layers[l][0][a][0] * scale) for a in agents]) for l in range(n_layers)])
        last_want = np.zeros_like(q_full)
        for sh, pool, ad in shards:
            cols = slice(sh.q_begin * dh, (sh.q_begin + sh.n_q_local) * dh)
            last_want[:, :, cols] = pool.decode(ad, 0, n_layers, agents, n_q, np.ascontiguousarray(q_full[:, :, cols]))
        cols = slice(mine_sh.q_begin * dh, (mine_sh.q_begin + mine_sh.n_q_local) * dh)
        if step < 3:
            _, last_dev = mine_pool.decode_gather(mine_ad, gather, 0, n_layers, agents, n_q, q=np.ascontiguousarray(q_full[:, :, cols]),
                                                  want_host=False)
        else:                                      # the host path waits for the handshake itself
            got, last_dev = mine_pool.decode_gather(mine_ad, gather, 0, n_layers, agents, n_q, q=np.ascontiguousarray(q_full[:, :, cols]))
            same = bool(np.array_equal(got, last_want))
            report.append(("overlap-host", step, same, 0.0, ctx.last_kernel()))
            ok = ok and same
        if step == 2:
            gather.wait()
            got_dev = np.zeros_like(last_want)
            ctx.d2h(got_dev, last_dev)
            ctx.synchronize()
            same = bool(np.array_equal(got_dev, last_want))
            report.append(("overlap-device", step, same, 0.0, ctx.last_kernel()))
            ok = ok and same
    gather.set_overlap(False)
    ok = ok and gather.steps() == 2 * steps + 4
    gather.check()
    # tear-down order of CUDA IPC: unmap the peers, barrier, free
    gather.disconnect()
    _barrier(d, "unmapped", rank, world)
    gather.close()
    _publish(os.path.join(d, f"result_{rank}"), repr((ok, report)).encode())
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main(int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else "gather"))
