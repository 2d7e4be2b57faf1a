"""The HBM-bound decode kernel (fla_decode_tma: TMA bulk-copy rings + tensor-core MMA over swizzled
bf16 pages) against the CPU oracle, through the C ABI.  Oracle = gqa_attention per (agent, layer)
(attention.hpp:332-363), which is what engine.hpp:440-443 calls once per agent per layer; inputs are
rounded to bf16 on the host and the oracle consumes the rounded values (tolerance 2e-2 on
max_rel_error, BASELINE.json north_star).  Needs a B200."""
import numpy as np
import pytest

from tests.test_gpu_pool import build_pool

pytestmark = pytest.mark.gpu

TOL = 2e-2


@pytest.fixture(scope="module")
def ctx():
    from paper_2602_01053_b200 import Context
    c = Context(0)
    yield c
    c.close()


def check_decode(ctx, orc, pool, ad, layers, batch, n_q, n_kv, L):
    """policy 0 = auto (mma.sync streaming kernel up to 32 rows per kv head, tcgen05 kernel in decode mode for
    33..128 rows), 2 = streaming kernel for every row count, 1 = CUDA cores."""
    n_layers = len(layers)
    rows = len(batch) * (n_q // n_kv)
    qs = np.stack([np.stack([layers[l][0][a][0] for a in batch]) for l in range(n_layers)])
    outs = {}
    for policy in (0, 2, 1):
        ctx.set_kernel_policy(policy)
        out = pool.decode(ad, 0, n_layers, batch, n_q, qs)
        outs[policy] = out
        want_kernel = {0: "fla_decode_umma" if 32 < rows <= 128 else "fla_decode_tma", 2: "fla_decode_tma",
                       1: "fla_paged_simt"}[policy]
        assert ctx.last_kernel() == want_kernel, (policy, rows, ctx.last_kernel())
        for l in range(n_layers):
            q, k, v, v_lr, b, s = layers[l]
            for i, a in enumerate(batch):
                bb = b[a] if len(b) else np.zeros((0, k.shape[1]), np.float32)
                want = orc.gqa_attention(q[a], k, v, v_lr, bb, s, L - 1, n_q, n_kv)
                err = orc.max_rel_error(out[l, i][None, :], want)
                assert err <= TOL, (policy, l, i, a, err, ctx.last_kernel())
    ctx.set_kernel_policy(0)
    # the kernel families agree far tighter than any of them agrees with the fp32 oracle's tolerance
    for pol in (0, 2):
        assert orc.max_rel_error(outs[pol].reshape(1, -1), outs[1].reshape(1, -1)) <= 1e-2


# n_q, n_kv, d, r, agents, L, P, layers  -- rows per kv head = agents * n_q / n_kv
SHAPES = [
    (8, 2, 128, 16, 3, 1000, 64, 2),    # 12 rows: one warp per worker (the Llama cfg-2 row count)
    (32, 8, 128, 16, 3, 257, 64, 1),    # Llama head counts
    (8, 2, 128, 64, 8, 777, 32, 1),     # 32 rows, rank 64: two warps per worker (the Mistral cfg-4 rows)
    (4, 1, 128, 32, 16, 530, 64, 1),    # 64 rows, rank 32: four warps per worker (cfg 5)
    (16, 2, 64, 8, 12, 300, 16, 1),     # 96 rows, d = 64, rank 8: eight warps per worker
    (8, 1, 128, 4, 20, 211, 16, 1),     # 160 rows: two 128-row blocks; rank 4 padded to 16
    (4, 1, 128, 16, 32, 1500, 64, 2),   # 128 rows exactly, 2 layers, a dozen key tiles per unit
    (8, 2, 64, 32, 10, 90, 32, 1),      # 40 rows, d = 64, a single (partial) key tile
    (4, 2, 64, 24, 2, 130, 128, 3),     # rank 24 padded to 32, 128-token pages, 3 layers
    (4, 2, 128, 2, 2, 48, 16, 1),       # rank 2 padded to 8
]


@pytest.mark.parametrize("n_q,n_kv,d,r,A,L,P,n_layers", SHAPES)
def test_decode_tma_matches_reference_path(ctx, orc, n_q, n_kv, d, r, A, L, P, n_layers):
    from paper_2602_01053_b200 import abi
    pool, ad, layers = build_pool(ctx, orc, "BaseLRShared", abi.BF16, 1000 + L, L, n_layers, n_q, n_kv, d, r, A, P=P)
    check_decode(ctx, orc, pool, ad, layers, list(range(A)), n_q, n_kv, L)
    pool.close()


@pytest.mark.parametrize("L", [1, 15, 16, 17, 31, 33, 64, 65, 4099])
def test_decode_tma_ragged_lengths(ctx, orc, L):
    """Single-token caches, tiles and pages that end mid-way; keys >= L must contribute exactly 0."""
    from paper_2602_01053_b200 import abi
    n_q, n_kv, d, r, A = 8, 2, 128, 16, 3
    pool, ad, layers = build_pool(ctx, orc, "BaseLRShared", abi.BF16, 50 + L, L, 1, n_q, n_kv, d, r, A, P=32)
    check_decode(ctx, orc, pool, ad, layers, [2, 0, 1, 1], n_q, n_kv, L)
    pool.close()


def test_decode_tma_rank_zero_is_plain_attention(ctx, orc):
    """FullShared keeps no LR cache: r = 0 must reduce to plain causal attention (test_attention.cpp:266-272)."""
    from paper_2602_01053_b200 import abi
    n_q, n_kv, d, A, L = 8, 2, 128, 3, 500
    pool, ad, layers = build_pool(ctx, orc, "FullShared", abi.BF16, 77, L, 2, n_q, n_kv, d, 0, A)
    check_decode(ctx, orc, pool, ad, layers, [0, 1, 2], n_q, n_kv, L)
    pool.close()


def test_decode_tma_large_scores_stay_exact_in_softmax(ctx, orc):
    """fuzz.hpp:30,40-43 drives scores to several hundred (amp 25) to stress the running-max logic;
    the lazy-rescale path must survive the same (inputs bf16-exact, so only P rounding differs)."""
    from paper_2602_01053_b200 import Adapters, Pool, abi
    from tests.cases import synthetic_layer
    n_q, n_kv, d, r, A, L = 8, 2, 128, 16, 2, 700
    for amp in (5.0, 25.0):
        q, k, v, v_lr, b, s = synthetic_layer(orc, 9, L, 1, n_q, n_kv, d, r, A, amp=amp)
        rnd = orc.round_bf16
        q = [rnd(x) for x in q]; k, v, v_lr = rnd(k), rnd(v), rnd(v_lr); b = [rnd(x) for x in b]
        pool = Pool(ctx, "BaseLRShared", 1, n_kv, d, 64, r, A, max_tokens=L, dtype=abi.BF16)
        ad = Adapters(ctx, 1, A, 64, r, n_kv, d, dtype=abi.BF16)
        pool.append_tokens(L)
        pool.append_key(0, 0, 0, k); pool.append_value(0, 0, 0, v); pool.append_lr(0, 0, 0, v_lr)
        for a in range(A):
            ad.set_b(0, a, b[a], 16.0)
        out = pool.decode(ad, 0, 1, [0, 1], n_q, np.stack([q[0][0], q[1][0]])[None])
        assert ctx.last_kernel() == "fla_decode_tma"
        for a in range(A):
            want = orc.gqa_attention(q[a], k, v, v_lr, b[a], s, L - 1, n_q, n_kv)
            assert orc.max_rel_error(out[0, a][None, :], want) <= TOL, (amp, a)
        pool.close(); ad.close()


@pytest.mark.parametrize("d,r,P", [(128, 16, 64), (64, 64, 16), (32, 8, 32), (16, 4, 16), (8, 32, 64), (24, 3, 16), (192, 100, 32)])
def test_swizzled_pages_read_back_bit_exact(ctx, orc, d, r, P):
    """key_view / value_view / lr_view (kvcache.hpp:307-324) de-paginate the swizzled bf16 layout:
    what comes back is exactly the bf16 rounding of what was appended, at every append granularity."""
    from paper_2602_01053_b200 import Pool, abi
    n_kv, L = 2, 203
    rng = np.random.default_rng(d * 1000 + r)
    k = orc.round_bf16(rng.standard_normal((L, n_kv * d)).astype(np.float32))
    v = orc.round_bf16(rng.standard_normal((L, n_kv * d)).astype(np.float32))
    lr = orc.round_bf16(rng.standard_normal((L, r)).astype(np.float32))
    pool = Pool(ctx, "BaseLRShared", 1, n_kv, d, 64, r, 2, max_tokens=L, dtype=abi.BF16, page_tokens=P)
    pool.append_tokens(L)
    row = 0
    for n in (1, 7, 16, 50, 129):       # ragged appends crossing page boundaries
        pool.append_key(0, 0, row, k[row:row + n]); pool.append_value(0, 0, row, v[row:row + n])
        pool.append_lr(0, 0, row, lr[row:row + n])
        row += n
    assert row == L
    assert np.array_equal(pool.key_view(0, 0), k)
    assert np.array_equal(pool.value_view(0, 0), v)
    assert np.array_equal(pool.lr_view(0, 0), lr)
    pool.close()


def test_decode_tma_layer_chunks_keep_results(ctx, orc):
    """A launch whose low-rank cache exceeds the L2 budget walks the layers in equal chunks inside the kernel (so that a
    chunk's V_lr, shared by the kv heads of a layer, is served by L2).  The chunked path needs >= 4 kv heads and a few
    dozen tiles per worker and chunk, so the case is 12 layers x 4 kv heads x 40 000 tokens with the planning L2 shrunk to
    20 MB (15.4 MB of V_lr: three chunks of four layers).  Chunking only changes which worker computes which (unit, tile)
    range, so the result must agree with the unchunked launch to split-merge rounding and with the reference path to the
    bf16 tolerance."""
    from paper_2602_01053_b200 import abi
    n_layers, n_q, n_kv, d, r, A, L = 12, 4, 4, 64, 16, 3, 40000
    pool, ad, layers = build_pool(ctx, orc, "BaseLRShared", abi.BF16, 3100, L, n_layers, n_q, n_kv, d, r, A)
    qs = np.stack([np.stack([layers[l][0][a][0] for a in range(A)]) for l in range(n_layers)])
    whole = pool.decode(ad, 0, n_layers, list(range(A)), n_q, qs)
    assert ctx.last_kernel() == "fla_decode_tma"
    ctx.set_l2_bytes(20 << 20)
    try:
        chunked = pool.decode(ad, 0, n_layers, list(range(A)), n_q, qs)
        assert ctx.last_kernel() == "fla_decode_tma (layer chunks)"
    finally:
        ctx.set_l2_bytes(126 << 20)
    assert orc.max_rel_error(chunked.reshape(1, -1), whole.reshape(1, -1)) <= 5e-3
    for l in (0, 3, 4, 11):                       # first and last layer of a chunk
        q, k, v, v_lr, b, s = layers[l]
        for a in range(A):
            want = orc.gqa_attention(q[a], k, v, v_lr, b[a], s, L - 1, n_q, n_kv)
            assert orc.max_rel_error(chunked[l, a][None, :], want) <= TOL, (l, a)
    pool.close()


def test_kernel_timing_api_averages_back_to_back_calls(ctx, orc):
    """lorakv_ctx_mean_kernel_ms: one event pair per fast-path call since profiling was switched on, no synchronisation
    between the calls (bench.py's roofline denominator)."""
    from paper_2602_01053_b200 import abi
    n_q, n_kv, d, r, A, L = 8, 2, 128, 16, 3, 2048
    pool, ad, layers = build_pool(ctx, orc, "BaseLRShared", abi.BF16, 5, L, 1, n_q, n_kv, d, r, A)
    qs = np.stack([layers[0][0][a][0] for a in range(A)])[None]
    ctx.set_profiling(True)
    with pytest.raises(abi.LorakvError, match="no profiled"):
        ctx.mean_kernel_ms()
    for _ in range(3):
        pool.decode(ad, 0, 1, list(range(A)), n_q, qs)
    ms, n = ctx.mean_kernel_ms()
    assert n == 3 and 0.0 < ms < 5.0
    assert 0.0 < ctx.last_kernel_ms() < 5.0
    pool.decode(ad, 0, 1, list(range(A)), n_q, qs)
    ms, n = ctx.mean_kernel_ms()             # the counter restarts after a read
    assert n == 1
    ctx.set_profiling(False)
    pool.close()
