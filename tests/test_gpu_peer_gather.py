"""The end-of-step output gather over peer memory (csrc/peer_gather.cu): the decode epilogue stores every
finished row into the gather buffer of every rank and a handshake kernel publishes the step.  Two ranks are two
PROCESSES here, both on cuda:0 (the box has one GPU): the buffers cross process boundaries through CUDA IPC exactly as
they do between GPUs.  The gathered rows must equal the shards' own outputs side by side BIT FOR BIT -- head shards
never interact (attention.hpp:347-361) -- and the reference path within the bf16 tolerance."""
import ast
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def ctx():
    from paper_2602_01053_b200 import Context
    c = Context(0)
    yield c
    c.close()


def test_single_rank_gather_is_the_plain_decode(ctx, orc):
    from paper_2602_01053_b200 import Gather, abi
    from tests.test_gpu_pool import build_pool
    n_q, n_kv, d, r, A, L, n_layers = 8, 2, 128, 16, 3, 700, 2
    pool, ad, layers = build_pool(ctx, orc, "BaseLRShared", abi.BF16, 77, L, n_layers, n_q, n_kv, d, r, A)
    qs = np.stack([np.stack([layers[l][0][a][0] for a in range(A)]) for l in range(n_layers)])
    g = Gather(ctx, 0, 1, qs.size)
    for policy in (0, 1):
        ctx.set_kernel_policy(policy)
        want = pool.decode(ad, 0, n_layers, list(range(A)), n_q, qs)
        for _ in range(3):      # both buffers of the pair
            got, dev = pool.decode_gather(ad, g, 0, n_layers, list(range(A)), n_q, q=qs)
            assert np.array_equal(got, want) and dev
    ctx.set_kernel_policy(0)
    assert g.steps() == 6
    with pytest.raises(abi.LorakvError, match="output floats"):
        pool.decode_gather(ad, g, 0, 1, list(range(A)), n_q, q=qs[:1])
    g.close(); pool.close()


def test_gather_argument_errors(ctx):
    from paper_2602_01053_b200 import Gather, abi
    with pytest.raises(abi.LorakvError, match="world size"):
        Gather(ctx, 0, 9, 16)
    with pytest.raises(abi.LorakvError, match="rank"):
        Gather(ctx, 2, 2, 16)
    g = Gather(ctx, 0, 2, 16)
    assert len(g.export()) == Gather.HANDLE_BYTES
    with pytest.raises(abi.LorakvError, match="handle bytes"):
        g.connect(b"\0" * 64)
    g.close()


def test_two_process_gather_over_cuda_ipc(tmp_path):
    world = 2
    env = dict(os.environ, PYTHONPATH=ROOT)
    procs = [subprocess.Popen([sys.executable, "-m", "tests.peer_gather_worker", str(r), str(world), str(tmp_path)], cwd=ROOT,
                              env=env, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True) for r in range(world)]
    outs = []
    try:
        for p in procs:
            outs.append(p.communicate(timeout=420)[0])
    finally:
        for p in procs:
            if p.poll() is None:
                p.kill()
    for r, p in enumerate(procs):
        assert p.returncode == 0, f"rank {r} failed:\n{outs[r][-3000:]}"
        ok, report = ast.literal_eval((tmp_path / f"result_{r}").read_text())
        assert ok, report
        kernels = {row[4] for row in report}
        assert kernels == {"fla_decode_tma", "fla_paged_simt"}, kernels
        assert all(row[2] for row in report), report           # bit-exact assembly on every step
        assert {row[0] for row in report} >= {0, 1, "overlap-device", "overlap-host"}      # incl. the overlapped handshake


def test_handshake_times_out_instead_of_hanging(tmp_path):
    """A peer that never issues the step: gather_sync_kernel gives up after lorakv_gather_set_timeout_ms, the call fails
    naming the step, lorakv_gather_check keeps failing -- the stream is never left spinning."""
    world = 2
    env = dict(os.environ, PYTHONPATH=ROOT)
    procs = [subprocess.Popen([sys.executable, "-m", "tests.peer_gather_worker", str(r), str(world), str(tmp_path), "timeout"], cwd=ROOT,
                              env=env, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True) for r in range(world)]
    outs = []
    try:
        for p in procs:
            outs.append(p.communicate(timeout=300)[0])
    finally:
        for p in procs:
            if p.poll() is None:
                p.kill()
    for r, p in enumerate(procs):
        assert p.returncode == 0, f"rank {r} failed:\n{outs[r][-3000:]}"
    ok, report = ast.literal_eval((tmp_path / "result_0").read_text())
    assert ok and "never published step 1" in report[0], report
