"""The tcgen05 prefill kernel (fla_prefill_umma: TMEM accumulators, TMA-staged swizzled pages) against
the CPU oracle through the C ABI.  Oracle = gqa_attention with L_c query rows at query_offset
(attention.hpp:332-363 as engine.hpp:440-443 calls it in prefill); inputs bf16-rounded on the host,
tolerance 2e-2 on max_rel_error (BASELINE.json north_star).  Needs a B200."""
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


def run_prefill(ctx, orc, n_q, n_kv, d, r, L, L_c, offsets, P, seed, scheme="BaseLRShared", amp=1.0, agent=1):
    from paper_2602_01053_b200 import abi
    A = 2
    pool, ad, layers = build_pool(ctx, orc, scheme, abi.BF16, seed, L, 1, n_q, n_kv, d, r, A, P=P)
    _, k, v, v_lr, b, s = layers[0]
    q = orc.round_bf16(orc.gaussian(L_c, n_q * d, seed + 77, amp / np.sqrt(d), np.float32))
    bb = b[agent] if r > 0 else np.zeros((0, n_kv * d), np.float32)
    for off in offsets:
        ctx.set_kernel_policy(0)
        got = pool.prefill(ad, 0, agent, n_q, q, off)
        assert ctx.last_kernel() == "fla_prefill_umma"
        want = orc.gqa_attention(q, k, v, v_lr, bb, s, off, n_q, n_kv)
        err = orc.max_rel_error(got, want)
        assert err <= TOL, (off, err)
        ctx.set_kernel_policy(1)
        ref = pool.prefill(ad, 0, agent, n_q, q, off)
        assert ctx.last_kernel() == "fla_paged_simt"
        ctx.set_kernel_policy(0)
        assert orc.max_rel_error(got, ref) <= 1e-2
    pool.close()


# n_q, n_kv, d, r, L, L_c, offsets, P
SHAPES = [
    (8, 2, 128, 16, 300, 40, (260, 0, 131), 64),       # group 4 -> 32 positions per CTA (the Llama mapping)
    (4, 2, 64, 8, 333, 77, (256, 100, 0), 64),          # d = 64, rank 8 padded to 16, group 2
    (4, 4, 128, 32, 700, 300, (400, 0), 32),            # group 1: 128 positions per CTA, rank 32, 32-token pages
    (16, 2, 128, 64, 520, 130, (390, 17), 128),         # group 8, rank 64, 128-token pages
    (8, 2, 128, 0, 450, 64, (386, 0), 16),              # rank 0 (FullShared), 16-token pages
    (32, 8, 128, 16, 1100, 96, (1004, 500), 64),        # Llama head counts; several key tiles
    (8, 2, 128, 16, 129, 2, (127, 0), 256),             # two query rows, 256-token pages
]


@pytest.mark.parametrize("n_q,n_kv,d,r,L,L_c,offsets,P", SHAPES)
def test_prefill_umma_matches_reference_path(ctx, orc, n_q, n_kv, d, r, L, L_c, offsets, P):
    run_prefill(ctx, orc, n_q, n_kv, d, r, L, L_c, offsets, P, seed=500 + L,
                scheme="FullShared" if r == 0 else "BaseLRShared")


def test_prefill_umma_large_scores(ctx, orc):
    """fuzz.hpp amplitudes (scores of several hundred) through the lazy-rescale / running-max logic."""
    for amp in (5.0, 25.0):
        from paper_2602_01053_b200 import Adapters, Pool, abi
        from tests.cases import synthetic_layer
        n_q, n_kv, d, r, L, L_c = 8, 2, 128, 16, 600, 200
        q1, k, v, v_lr, b, s = synthetic_layer(orc, 21, L, 1, n_q, n_kv, d, r, 2, amp=amp)
        rnd = orc.round_bf16
        k, v, v_lr = rnd(k), rnd(v), rnd(v_lr); b = [rnd(x) for x in b]
        q = rnd(orc.gaussian(L_c, n_q * d, 4321, amp / np.sqrt(d), np.float32))
        pool = Pool(ctx, "BaseLRShared", 1, n_kv, d, 64, r, 2, max_tokens=L, dtype=abi.BF16)
        ad = Adapters(ctx, 1, 2, 64, r, n_kv, d, dtype=abi.BF16)
        pool.append_tokens(L)
        pool.append_key(0, 0, 0, k); pool.append_value(0, 0, 0, v); pool.append_lr(0, 0, 0, v_lr)
        for a in range(2):
            ad.set_b(0, a, b[a], 16.0)
        got = pool.prefill(ad, 0, 0, n_q, q, L - L_c)
        assert ctx.last_kernel() == "fla_prefill_umma"
        want = orc.gqa_attention(q, k, v, v_lr, b[0], s, L - L_c, n_q, n_kv)
        assert orc.max_rel_error(got, want) <= TOL, amp
        pool.close(); ad.close()


def test_prefill_umma_masked_keys_contribute_exactly_zero(ctx, orc):
    """test_attention.cpp:144-175 through the paged prefill: keys beyond every row's causal boundary hold
    1e6-sized values and must not change a single bit of the output."""
    from paper_2602_01053_b200 import Adapters, Pool, abi
    from tests.cases import synthetic_layer
    n_q, n_kv, d, r, L, L_c, off = 8, 2, 128, 16, 400, 50, 100       # rows see keys <= 149; 150..399 are hidden
    _, k, v, v_lr, b, s = synthetic_layer(orc, 33, L, 1, n_q, n_kv, d, r, 2)
    rnd = orc.round_bf16
    k, v, v_lr = rnd(k), rnd(v), rnd(v_lr); b = [rnd(x) for x in b]
    q = rnd(orc.gaussian(L_c, n_q * d, 99, 1.0 / np.sqrt(d), np.float32))
    outs = []
    for poison in (False, True):
        kk, vv, ll = k.copy(), v.copy(), v_lr.copy()
        if poison:
            kk[off + L_c:] = 1e6; vv[off + L_c:] = -1e6; ll[off + L_c:] = 1e6
        pool = Pool(ctx, "BaseLRShared", 1, n_kv, d, 64, r, 2, max_tokens=L, dtype=abi.BF16)
        ad = Adapters(ctx, 1, 2, 64, r, n_kv, d, dtype=abi.BF16)
        pool.append_tokens(L)
        pool.append_key(0, 0, 0, kk); pool.append_value(0, 0, 0, vv); pool.append_lr(0, 0, 0, ll)
        for a in range(2):
            ad.set_b(0, a, b[a], 16.0)
        outs.append(pool.prefill(ad, 0, 1, n_q, q, off))
        assert ctx.last_kernel() == "fla_prefill_umma"
        pool.close(); ad.close()
    assert np.array_equal(outs[0], outs[1])
