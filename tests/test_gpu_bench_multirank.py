"""The N > 1 flow of bench.py end to end on a one-GPU box: two ranks (torchrun) share cuda:0 over a gloo rendezvous
(LORAKV_BENCH_SHARE_GPU=1 -- NCCL refuses two ranks on one device), each holding one kv-head shard, the end-of-step
output gather going through the peer-memory path (csrc/peer_gather.cu) and checked bit for bit against slab + all_gather
inside the bench.  Timings of such a run mean nothing; the JSON contract and the gather are what is tested."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("gather", ["peer", "nccl"])
def test_two_rank_bench_line(gather):
    env = dict(os.environ, LORAKV_BENCH_SHARE_GPU="1", PYTHONPATH=ROOT)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr", "127.0.0.1",
           "--master-port", str(_free_port()), os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "4", "--warmup", "3",
           "--workload", "cfg1", "--gather", gather]
    res = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, (res.stdout + res.stderr)[-3000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, res.stdout[-2000:]            # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["workload"] == "cfg1" and d["config"]["parallelism"] == "kv-head shard x2"
    assert d["gpu_launches"] > 0 and d["value"] > 0 and d["e2e"]["value"] > 0
    assert d["e2e"]["d2h_bytes_per_step"] == 2 * d["e2e"]["h2d_bytes_per_step"]      # every rank reads the gathered rows back
    # the cost of the end-of-step gather per mode, and every rank's own kernel / step time
    comm = d["comm"]
    assert [r["rank"] for r in comm["per_rank"]] == [0, 1] and all(r["kernel_ms"] > 0 and r["step_ms"] > 0 for r in comm["per_rank"])
    assert comm["attention_only_ms"] > 0 and comm["nccl_all_gather"]["step_ms"] > 0 and comm["bytes_per_rank"] > 0
    assert (comm["peer_memory"]["step_ms"] is not None) == (gather == "peer")
    if gather == "peer":
        assert d["config"]["output_gather"] == "peer"
        assert d["config"]["output_gather_check"] == "bit-exact vs all_gather on every rank"
    else:
        assert d["config"]["output_gather"] == "nccl"
