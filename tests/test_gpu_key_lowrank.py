"""The key-side low-rank term of the north star: S = (q K_base^T + (k_scale q B_k^T) L_k^T) / sqrt(d), i.e. attention over the
effective keys K_eff = K_base + k_scale * L_k B_k WITHOUT forming them (L_k = X A_k is one L x r_k cache per layer, B_k is per
agent).

PARITY UNPINNED: the reference has no key adapter (proj/include/lorakv/engine.hpp:129-130, attention.hpp:47-56; the paper
rules it out under RoPE), so no reference test or golden vector covers it.  The checker here
materialises K_eff with the reference's own matmul and calls the reference's attention (naive_attention / gqa_attention,
attention.hpp:81, :332) on it; r_k = 0 must reproduce the reference path bit for bit."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    import paper_2602_01053_b200 as pkg
    c = pkg.Context(0)
    yield c
    c.close()


def k_eff(orc, k, l_k, b_k, k_scale):
    return (k + np.asarray(k_scale, dtype=k.dtype) * orc.matmul(l_k, b_k)).astype(k.dtype)


@pytest.mark.parametrize("dtype,tol", [(np.float64, 1e-10), (np.float32, 1e-4)])
@pytest.mark.parametrize("L,L_c,n_q,n_kv,d,r,r_k", [(37, 1, 1, 1, 16, 2, 3), (64, 9, 4, 2, 64, 8, 8), (50, 50, 6, 3, 4, 0, 1), (33, 5, 2, 2, 32, 1, 16)])
def test_generic_operator_against_materialised_keys(ctx, orc, dtype, tol, L, L_c, n_q, n_kv, d, r, r_k):
    g = lambda rows, cols, key, scale: orc.gaussian(rows, cols, orc.child(991 + L, key), scale, dtype)
    q, k, v = g(L_c, n_q * d, 1, d ** -0.5), g(L, n_kv * d, 2, d ** -0.5), g(L, n_kv * d, 3, 1.0)
    v_lr, b_up = g(L, r, 4, 1.0), g(r, n_kv * d, 5, 0.3)
    l_k, b_k = g(L, r_k, 6, 1.0), g(r_k, n_kv * d, 7, 0.3 * d ** -0.5)
    off = L - L_c
    want = orc.gqa_attention(q, k_eff(orc, k, l_k, b_k, 0.5), v, v_lr, b_up, 0.25, off, n_q, n_kv)
    got = ctx.gqa_attention_keylr(q, k, v, v_lr, b_up, 0.25, l_k, b_k, 0.5, off, n_q, n_kv)
    assert orc.max_rel_error(got, want) <= tol
    # the adapter must matter in this case (otherwise the test proves nothing) ...
    assert orc.max_rel_error(ctx.gqa_attention(q, k, v, v_lr, b_up, 0.25, off, n_q, n_kv), want) > 100 * tol
    # ... and r_k = 0 is the reference operator, bit for bit
    none = ctx.gqa_attention_keylr(q, k, v, v_lr, b_up, 0.25, l_k[:, :0], b_k[:0], 0.5, off, n_q, n_kv)
    assert np.array_equal(none, ctx.gqa_attention(q, k, v, v_lr, b_up, 0.25, off, n_q, n_kv))


def build(ctx, orc, dtype_name, scheme, n_layers, L, n_q, n_kv, d, r, r_k, A, d_model, seed, P=32):
    from paper_2602_01053_b200 import Adapters, Pool, abi
    dt = abi.BF16 if dtype_name == "bf16" else abi.F32
    rnd = orc.round_bf16 if dtype_name == "bf16" else (lambda a: a)
    g = lambda rows, cols, key, scale: rnd(orc.gaussian(rows, cols, orc.child(seed, key), scale, np.float32))
    pool = Pool(ctx, scheme, n_layers, n_kv, d, d_model, r, A, max_tokens=L, dtype=dt, page_tokens=P, rank_k=r_k)
    ad = Adapters(ctx, n_layers, A, d_model, max(r, 1), n_kv, d, dtype=dt)
    ad.enable_key(r_k)
    pool.append_tokens(L)
    layers = []
    for l in range(n_layers):
        x = g(L, d_model, 100 * l + 1, 1.0)
        k, v = g(L, n_kv * d, 100 * l + 2, d ** -0.5), g(L, n_kv * d, 100 * l + 3, 1.0)
        a_v, a_k = g(d_model, max(r, 1), 100 * l + 4, d_model ** -0.5), g(d_model, r_k, 100 * l + 5, d_model ** -0.5)
        b_v = [g(max(r, 1), n_kv * d, 100 * l + 10 + a, 0.02 / np.sqrt(max(r, 1))) for a in range(A)]
        b_k = [g(r_k, n_kv * d, 100 * l + 20 + a, 1.5 * d ** -0.5) for a in range(A)]
        pool.append_key(l, 0, 0, k); pool.append_value(l, 0, 0, v)
        ad.set_a(l, a_v); ad.set_a_k(l, a_k)
        for a in range(A):
            ad.set_b(l, a, b_v[a], 16.0); ad.set_b_k(l, a, b_k[a], 64.0)
        if r > 0:
            assert pool.append_lr_project(ad, l, 0, 0, x) == L
        assert pool.append_lk_project(ad, l, 0, x) == L
        v_lr = pool.lr_view(l, 0) if r > 0 else np.zeros((L, 0), np.float32)      # the rows the cache holds (bf16-rounded X A)
        l_k = pool.lk_view(l)
        assert orc.max_rel_error(l_k, orc.matmul(x, a_k)) <= (4e-3 if dtype_name == "bf16" else 1e-5)
        layers.append(dict(k=k, v=v, v_lr=v_lr, l_k=l_k, b_v=[b[:r] for b in b_v] if r > 0 else [np.zeros((0, n_kv * d), np.float32)] * A, b_k=b_k))
    return pool, ad, layers, g


@pytest.mark.parametrize("dtype_name,tol", [("f32", 1e-4), ("bf16", 2e-2)])
@pytest.mark.parametrize("n_q,n_kv,d,r,r_k,A,L", [(8, 2, 128, 16, 16, 3, 200), (4, 2, 64, 8, 8, 2, 150), (8, 2, 128, 0, 32, 2, 96), (32, 8, 128, 16, 16, 3, 700)])
def test_paged_decode_and_prefill_with_the_key_term(ctx, orc, dtype_name, tol, n_q, n_kv, d, r, r_k, A, L):
    n_layers, d_model = 2, 128
    pool, ad, layers, g = build(ctx, orc, dtype_name, "BaseLRShared" if r > 0 else "FullShared", n_layers, L, n_q, n_kv, d, r, r_k, A, d_model, 4100 + L)
    q = np.stack([np.stack([g(1, n_q * d, 7000 + 10 * l + a, d ** -0.5)[0] for a in range(A)]) for l in range(n_layers)])
    out = pool.decode(ad, 0, n_layers, list(range(A)), n_q, q)
    kernel = ctx.last_kernel()
    # bf16 pages with <= 16 query rows per kv head: the TMA / tensor-core decode kernel carries the term (one more k block of
    # the score MMA); everything else runs on the CUDA-core paged kernel
    assert kernel == ("fla_decode_tma" if dtype_name == "bf16" else "fla_paged_simt")
    ctx.set_kernel_policy(1)
    try:
        cross = pool.decode(ad, 0, n_layers, list(range(A)), n_q, q)
        assert ctx.last_kernel() == "fla_paged_simt"
    finally:
        ctx.set_kernel_policy(0)
    assert orc.max_rel_error(out.reshape(1, -1), cross.reshape(1, -1)) <= tol
    for l in range(n_layers):
        lay = layers[l]
        for a in range(A):
            keys = k_eff(orc, lay["k"], lay["l_k"], lay["b_k"][a], 64.0 / r_k)
            want = orc.gqa_attention(q[l, a][None, :], keys, lay["v"], lay["v_lr"], lay["b_v"][a], 16.0 / max(r, 1), L - 1, n_q, n_kv)
            assert orc.max_rel_error(out[l, a][None, :], want) <= tol, (l, a, kernel)
            plain = orc.gqa_attention(q[l, a][None, :], lay["k"], lay["v"], lay["v_lr"], lay["b_v"][a], 16.0 / max(r, 1), L - 1, n_q, n_kv)
            assert orc.max_rel_error(plain, want) > 2 * tol                        # the key adapter matters here
    # a prefill block of one agent (causal mask inside the block)
    L_c = 24
    qb = g(L_c, n_q * d, 8000, d ** -0.5)
    got = pool.prefill(ad, 1, 1, n_q, qb, L - L_c)
    assert ctx.last_kernel() == ("fla_prefill_umma" if dtype_name == "bf16" else "fla_paged_simt")
    lay = layers[1]
    want = orc.gqa_attention(qb, k_eff(orc, lay["k"], lay["l_k"], lay["b_k"][1], 64.0 / r_k), lay["v"], lay["v_lr"], lay["b_v"][1],
                             16.0 / max(r, 1), L - L_c, n_q, n_kv)
    assert orc.max_rel_error(got, want) <= tol
    pool.close(); ad.close()


@pytest.mark.parametrize("n_q,n_kv,d,r,r_k,A,L,P,want_kernel", [
    (32, 8, 128, 16, 16, 12, 900, 32, "umma"),      # 48 rows per kv head: the tcgen05 kernel in decode mode
    (16, 4, 128, 16, 16, 6, 640, 32, "umma"),       # 24 rows per kv head: beyond the streaming kernel's 16, tcgen05 decode mode
    (16, 4, 128, 32, 32, 9, 1500, 64, "umma"),      # two k steps of the key term, SWIZZLE_64B tiles, two-stage rings
    (8, 2, 64, 64, 20, 10, 700, 16, "umma"),        # d_head 64 leaves TMEM columns even beside a rank-64 value side
    (16, 4, 128, 0, 8, 9, 333, 128, "umma"),        # no value-side cache at all
    (16, 4, 128, 64, 16, 9, 300, 32, "simt"),       # d_head 128 + rank 64: no room for Qk in TMEM -> CUDA-core kernel
])
def test_key_term_on_the_tcgen05_kernels(ctx, orc, n_q, n_kv, d, r, r_k, A, L, P, want_kernel):
    """Prefill blocks and wide decode batches with the key-side term on fla_prefill_umma / fla_decode_umma: L_k tiles ride in the
    K stage, Qk = k_scale q B_k^T sits in TMEM beside Q, the score chain takes rank_k / 16 more k steps."""
    tol = 2e-2
    n_layers, d_model = 2, 128
    pool, ad, layers, g = build(ctx, orc, "bf16", "BaseLRShared" if r > 0 else "FullShared", n_layers, L, n_q, n_kv, d, r, r_k, A, d_model,
                                5200 + L, P=P)
    q = np.stack([np.stack([g(1, n_q * d, 7000 + 10 * l + a, d ** -0.5)[0] for a in range(A)]) for l in range(n_layers)])
    out = pool.decode(ad, 0, n_layers, list(range(A)), n_q, q)
    assert ctx.last_kernel() == ("fla_decode_umma" if want_kernel == "umma" else "fla_paged_simt")
    for l in range(n_layers):
        lay = layers[l]
        for a in (0, A // 2, A - 1):
            keys = k_eff(orc, lay["k"], lay["l_k"], lay["b_k"][a], 64.0 / r_k)
            want = orc.gqa_attention(q[l, a][None, :], keys, lay["v"], lay["v_lr"], lay["b_v"][a], 16.0 / max(r, 1), L - 1, n_q, n_kv)
            assert orc.max_rel_error(out[l, a][None, :], want) <= tol, (l, a)
            plain = orc.gqa_attention(q[l, a][None, :], lay["k"], lay["v"], lay["v_lr"], lay["b_v"][a], 16.0 / max(r, 1), L - 1, n_q, n_kv)
            assert orc.max_rel_error(plain, want) > 2 * tol
    # prefill blocks: several 128-row CTAs per kv head, the block starting mid-page and ending at the last row
    for L_c, off in ((min(L, 200), L - min(L, 200)), (77, 13)):
        qb = g(L_c, n_q * d, 8000 + L_c, d ** -0.5)
        Lv = off + L_c                     # rows beyond the block are invisible (causal): the checker sees the prefix only
        got = pool.prefill(ad, 1, A - 1, n_q, qb, off)
        assert ctx.last_kernel() == ("fla_prefill_umma" if want_kernel == "umma" else "fla_paged_simt")
        lay = layers[1]
        want = orc.gqa_attention(qb, k_eff(orc, lay["k"], lay["l_k"], lay["b_k"][A - 1], 64.0 / r_k)[:Lv], lay["v"][:Lv], lay["v_lr"][:Lv],
                                 lay["b_v"][A - 1], 16.0 / max(r, 1), off, n_q, n_kv)
        assert orc.max_rel_error(got, want) <= tol
        ctx.set_kernel_policy(1)
        try:
            cross = pool.prefill(ad, 1, A - 1, n_q, qb, off)
        finally:
            ctx.set_kernel_policy(0)
        assert orc.max_rel_error(got, cross) <= tol
    pool.close(); ad.close()


def test_key_cache_bookkeeping_and_errors(ctx, orc):
    from paper_2602_01053_b200 import Adapters, Pool, abi
    n_kv, d, r, r_k, A, d_model, L = 2, 64, 8, 4, 2, 64, 40
    pool = Pool(ctx, "BaseLRShared", 1, n_kv, d, d_model, r, A, max_tokens=64, dtype=abi.F32, page_tokens=16, rank_k=r_k)
    plain = Pool(ctx, "BaseLRShared", 1, n_kv, d, d_model, r, A, max_tokens=64, dtype=abi.F32, page_tokens=16)
    ad = Adapters(ctx, 1, A, d_model, r, n_kv, d, dtype=abi.F32)
    rows = orc.gaussian(L, r_k, 5, 1.0, np.float32)
    pool.append_tokens(L)
    assert pool.append_lk(0, 0, rows[:25]) == 25 and pool.append_lk(0, 20, rows[20:]) == 15       # first writer wins
    assert np.array_equal(pool.lk_view(0), rows)
    with pytest.raises(abi.LorakvError, match="gap"):
        pool.append_lk(0, L + 3, rows[:2])
    with pytest.raises(abi.LorakvError, match="no key-side low-rank cache"):
        plain.append_lk(0, 0, rows)
    assert pool.bytes()["lr"] == L * r_k * 4                                     # L_k rows count as low-rank bytes
    assert list(pool.page_table(4, 0)) == [0, 1, 2]
    k = orc.gaussian(L, n_kv * d, 6, 1.0, np.float32)
    pool.append_key(0, 0, 0, k); pool.append_value(0, 0, 0, k); pool.append_lr(0, 0, 0, orc.gaussian(L, r, 7, 1.0, np.float32))
    ad.set_b(0, 0, np.zeros((r, n_kv * d), np.float32), 16.0)
    q = np.zeros((1, 1, 4 * d), np.float32)
    with pytest.raises(abi.LorakvError, match="key rank"):                        # tables without the key side
        pool.decode(ad, 0, 1, [0], 4, q)
    ad.enable_key(r_k)
    with pytest.raises(abi.LorakvError, match="B_k"):
        pool.decode(ad, 0, 1, [0], 4, q)
    pool.close(); plain.close(); ad.close()
