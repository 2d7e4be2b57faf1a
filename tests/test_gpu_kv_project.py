"""The projection that feeds the cache: K / V_base projection of new context rows, RoPE on the
keys and the append into the paged cache in one call, against the reference path restated by the oracle:
    k = matmul(x, Wk); apply_rope(k, n_kv, d, row_begin); v = matmul(x, Wv); append_key / append_value
(engine.hpp:376-403, :225-243; matmul matrix.hpp:101-111).  bf16 pools with d_head 128 run the tcgen05 kernel
(kv_project_umma), fp32 pools the reference's own summation order.  Needs a B200."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    from paper_2602_01053_b200 import Context
    c = Context(0)
    yield c
    c.close()


def reference_kv(orc, x, wk, wv, n_kv, d, row_begin, rope):
    k = orc.matmul(x, wk)
    if rope:
        k = orc.apply_rope(k, n_kv, d, row_begin)
    return k, orc.matmul(x, wv)


def make_inputs(orc, seed, L, d_model, n_kv, d, bf16):
    x = orc.gaussian(L, d_model, orc.child(seed, 1), 1.0, np.float32)
    wk = orc.gaussian(d_model, n_kv * d, orc.child(seed, 2), 1.0 / np.sqrt(d_model), np.float32)   # engine.hpp:152-153
    wv = orc.gaussian(d_model, n_kv * d, orc.child(seed, 3), 1.0 / np.sqrt(d_model), np.float32)
    if bf16:
        x, wk, wv = orc.round_bf16(x), orc.round_bf16(wk), orc.round_bf16(wv)
    return x, wk, wv


# L, d_model, n_kv, P, row chunks (appended one after the other, so later chunks start mid-page / mid-tile), rope
BF16_CASES = [
    (300, 256, 2, 64, (300,), True),
    (200, 192, 1, 32, (37, 100, 63), True),          # one kv head: a tile holds a K head and a V head
    (1000, 512, 4, 64, (128, 872), True),            # several 256-column blocks, a full first tile
    (130, 64, 2, 16, (130,), False),                 # single k block, no rotation
    (90, 4096, 2, 128, (90,), True),                 # the Llama reduction depth
]


@pytest.mark.parametrize("L,d_model,n_kv,P,chunks,rope", BF16_CASES)
def test_fused_projection_rope_append_bf16(ctx, orc, L, d_model, n_kv, P, chunks, rope):
    from paper_2602_01053_b200 import Pool, Projection, abi
    d = 128
    x, wk, wv = make_inputs(orc, 700 + L, L, d_model, n_kv, d, True)
    pool = Pool(ctx, "FullShared", 2, n_kv, d, d_model, 0, 1, max_tokens=L + 8, dtype=abi.BF16, page_tokens=P)
    proj = Projection(ctx, 2, d_model, n_kv, d, dtype=abi.BF16)
    proj.set_kv(1, wk, wv)
    pool.append_tokens(L)
    r0 = 0
    for n in chunks:
        assert pool.append_kv_project(proj, 1, 0, r0, x[r0:r0 + n], rope=rope) == n
        assert ctx.last_kernel() == "kv_project_umma"
        r0 += n
    assert pool.append_kv_project(proj, 1, 0, 0, x, rope=rope) == 0            # first writer wins: nothing to add
    want_k, want_v = reference_kv(orc, x, wk, wv, n_kv, d, 0, rope)
    got_k, got_v = pool.key_view(1, 0), pool.value_view(1, 0)
    assert got_k.shape == want_k.shape and got_v.shape == want_v.shape
    # bf16 storage of fp32-accumulated exact products: half a bf16 ulp (2^-9) of the largest element
    assert orc.max_rel_error(got_k, want_k) <= 4e-3
    assert orc.max_rel_error(got_v, want_v) <= 4e-3
    assert np.mean(got_v == orc.round_bf16(want_v)) > 0.97                       # the rest are 1-ulp rounding flips
    assert pool.rows(abi.KEY, 0, 0) == 0                                         # the other layer is untouched
    pool.close(); proj.close()


def test_fused_projection_then_attention_matches_reference_step(ctx, orc):
    """The hot path end to end on one layer: project + rotate + append K / V, project V_lr = X * A, then decode over
    the cache -- against gqa_attention on the reference's k / v / v_lr (engine.hpp:376-443)."""
    from paper_2602_01053_b200 import Adapters, Pool, Projection, abi
    L, d_model, n_q, n_kv, d, r, A = 333, 256, 8, 2, 128, 16, 2
    x, wk, wv = make_inputs(orc, 4242, L, d_model, n_kv, d, True)
    a = orc.round_bf16(orc.gaussian(d_model, r, orc.child(4242, 4), 1.0 / np.sqrt(d_model), np.float32))
    b = [orc.round_bf16(orc.gaussian(r, n_kv * d, orc.child(4242, 10 + i), 0.02 / np.sqrt(r), np.float32)) for i in range(A)]
    q = [orc.round_bf16(orc.gaussian(1, n_q * d, orc.child(4242, 20 + i), 1.0 / np.sqrt(d), np.float32)) for i in range(A)]
    pool = Pool(ctx, "BaseLRShared", 1, n_kv, d, d_model, r, A, max_tokens=L, dtype=abi.BF16)
    proj = Projection(ctx, 1, d_model, n_kv, d, dtype=abi.BF16)
    ad = Adapters(ctx, 1, A, d_model, r, n_kv, d, dtype=abi.BF16)
    proj.set_kv(0, wk, wv); ad.set_a(0, a)
    for i in range(A):
        ad.set_b(0, i, b[i], 16.0)
    pool.append_tokens(L)
    assert pool.append_kv_project(proj, 0, 0, 0, x) == L
    assert pool.append_lr_project(ad, 0, 0, 0, x) == L
    out = pool.decode(ad, 0, 1, list(range(A)), n_q, np.stack([q[i][0] for i in range(A)])[None])
    k, v = reference_kv(orc, x, wk, wv, n_kv, d, 0, True)
    v_lr = orc.matmul(x, a)
    for i in range(A):
        want = orc.gqa_attention(q[i], k, v, v_lr, b[i], 16.0 / r, L - 1, n_q, n_kv)
        assert orc.max_rel_error(out[0, i][None, :], want) <= 2e-2
    pool.close(); proj.close(); ad.close()


@pytest.mark.parametrize("d,n_kv,rope", [(32, 2, True), (128, 1, True), (64, 3, False)])
def test_projection_rope_append_fp32_is_the_reference_order(ctx, orc, d, n_kv, rope):
    """fp32 pools: matmul in the reference's order (bit-identical) and the rotation with double-precision angles."""
    from paper_2602_01053_b200 import Pool, Projection, abi
    L, d_model = 150, 96
    x, wk, wv = make_inputs(orc, 31 + d, L, d_model, n_kv, d, False)
    pool = Pool(ctx, "FullShared", 1, n_kv, d, d_model, 0, 1, max_tokens=L, dtype=abi.F32, page_tokens=32)
    proj = Projection(ctx, 1, d_model, n_kv, d, dtype=abi.F32)
    proj.set_kv(0, wk, wv)
    pool.append_tokens(L)
    assert pool.append_kv_project(proj, 0, 0, 0, x[:70], rope=rope) == 70
    assert pool.append_kv_project(proj, 0, 0, 40, x[40:], rope=rope) == L - 70       # overlaps 30 cached rows
    assert ctx.last_kernel() == "kv_project_f32"
    want_k, want_v = reference_kv(orc, x, wk, wv, n_kv, d, 0, rope)
    assert np.array_equal(pool.value_view(0, 0), want_v)
    assert orc.max_rel_error(pool.key_view(0, 0), want_k) <= 1e-6
    if not rope:
        assert np.array_equal(pool.key_view(0, 0), want_k)
    pool.close(); proj.close()


def test_projection_errors(ctx, orc):
    from paper_2602_01053_b200 import LorakvError, Pool, Projection, abi
    pool = Pool(ctx, "FullShared", 1, 2, 128, 64, 0, 1, max_tokens=64, dtype=abi.BF16)
    proj = Projection(ctx, 1, 64, 2, 128, dtype=abi.BF16)
    x = np.zeros((4, 64), np.float32)
    pool.append_tokens(8)
    with pytest.raises(LorakvError, match="never uploaded"):
        pool.append_kv_project(proj, 0, 0, 0, x)
    proj.set_kv(0, np.zeros((64, 256), np.float32), np.zeros((64, 256), np.float32))
    with pytest.raises(LorakvError, match="gap"):
        pool.append_kv_project(proj, 0, 0, 3, x)                                       # kvcache.hpp:401-403
    other = Projection(ctx, 1, 128, 2, 128, dtype=abi.BF16)
    with pytest.raises(LorakvError, match="do not match"):
        pool.append_kv_project(other, 0, 0, 0, x)
    pool.close(); proj.close(); other.close()


def reference_q(orc, x, wq, a, b, alpha, n_q, d, pos, rope):
    """engine.hpp:362-373, :422"""
    q = orc.matmul(x, wq)
    if a is not None:
        q = q + np.float32(alpha / a.shape[1]) * orc.matmul(orc.matmul(x, a), b)
    return orc.apply_rope(q, n_q, d, pos) if rope else q


@pytest.mark.parametrize("L,d_model,n_q,n_kv,r,pos,rope,shard", [
    (200, 256, 8, 2, 16, 37, True, None),
    (130, 192, 4, 2, 8, 0, True, None),
    (300, 512, 16, 4, 64, 1000, True, (2, 2)),      # this shard holds kv heads 2..3 -> q heads 8..15
    (77, 128, 4, 1, 2, 5, False, None),
])
def test_query_projection_with_q_lora_and_rope_bf16(ctx, orc, L, d_model, n_q, n_kv, r, pos, rope, shard):
    """q = rope(x Wq + (alpha/r) (x A_q) B_q[agent]) on the tcgen05 kernel (bf16 operands, fp32 accumulation and output)."""
    from paper_2602_01053_b200 import Projection, abi
    d, A = 128, 2
    x = orc.round_bf16(orc.gaussian(L, d_model, orc.child(L, 1), 1.0, np.float32))
    wq = orc.round_bf16(orc.gaussian(d_model, n_q * d, orc.child(L, 2), 1.0 / np.sqrt(d_model), np.float32))
    a = orc.round_bf16(orc.gaussian(d_model, r, orc.child(L, 3), 1.0 / np.sqrt(d_model), np.float32))
    b = [orc.round_bf16(orc.gaussian(r, n_q * d, orc.child(L, 10 + i), 0.02 / np.sqrt(r), np.float32)) for i in range(A)]
    kb, kn = shard if shard else (0, n_kv)
    proj = Projection(ctx, 1, d_model, n_kv, d, kv_head_begin=kb, n_kv_local=kn, dtype=abi.BF16)
    proj.set_q(0, n_q, wq)
    for i in range(A):
        proj.set_q_lora(0, i, A, a, b[i], 16.0)
    g = n_q // n_kv
    cols = slice(kb * g * d, (kb + kn) * g * d)
    for agent in (1, -1):
        got = proj.query(0, agent, pos, x, kn * g * d, rope=rope)
        assert ctx.last_kernel() == "q_project_umma"
        want = reference_q(orc, x, wq, a if agent >= 0 else None, b[agent] if agent >= 0 else None, 16.0, n_q, d, pos, rope)[:, cols]
        assert orc.max_rel_error(got, want) <= 1e-4, agent
    proj.close()


def test_query_projection_fp32_is_the_reference_order(ctx, orc):
    from paper_2602_01053_b200 import Projection, abi
    L, d_model, n_q, n_kv, d, r = 90, 96, 4, 2, 32, 4
    x = orc.gaussian(L, d_model, 1, 1.0, np.float32)
    wq = orc.gaussian(d_model, n_q * d, 2, 1.0 / np.sqrt(d_model), np.float32)
    a = orc.gaussian(d_model, r, 3, 1.0 / np.sqrt(d_model), np.float32)
    b = orc.gaussian(r, n_q * d, 4, 0.02 / np.sqrt(r), np.float32)
    proj = Projection(ctx, 1, d_model, n_kv, d, dtype=abi.F32)
    proj.set_q(0, n_q, wq)
    proj.set_q_lora(0, 0, 1, a, b, 16.0)
    got = proj.query(0, 0, 11, x, n_q * d, rope=False)
    assert ctx.last_kernel() == "q_project_f32"
    assert np.array_equal(got, reference_q(orc, x, wq, a, b, 16.0, n_q, d, 11, False))        # bit for bit
    got = proj.query(0, 0, 11, x, n_q * d, rope=True)
    assert orc.max_rel_error(got, reference_q(orc, x, wq, a, b, 16.0, n_q, d, 11, True)) <= 1e-6
    proj.close()


@pytest.mark.parametrize("dtype_name,d,scheme", [("BF16", 128, "NonShared"), ("BF16", 128, "FullShared"), ("F32", 32, "NonShared")])
def test_full_values_projection_merges_the_value_lora(ctx, orc, dtype_name, d, scheme):
    """NonShared / FullShared store v_base + (alpha/r) (x A_v) B_v[agent] (engine.hpp:385-393) and attend with r = 0."""
    from paper_2602_01053_b200 import Adapters, Pool, Projection, abi
    dtype = getattr(abi, dtype_name)
    bf16 = dtype == abi.BF16
    L, d_model, n_kv, r, A = 140, 128, 2, 8, 2
    x, wk, wv = make_inputs(orc, 9000 + d, L, d_model, n_kv, d, bf16)
    rnd = orc.round_bf16 if bf16 else (lambda m: m)
    a = rnd(orc.gaussian(d_model, r, orc.child(9000, 4), 1.0 / np.sqrt(d_model), np.float32))
    b = [rnd(orc.gaussian(r, n_kv * d, orc.child(9000, 10 + i), 0.02 / np.sqrt(r), np.float32)) for i in range(A)]
    pool = Pool(ctx, scheme, 1, n_kv, d, d_model, 0, A, max_tokens=L, dtype=dtype, page_tokens=32)
    proj = Projection(ctx, 1, d_model, n_kv, d, dtype=dtype)
    ad = Adapters(ctx, 1, A, d_model, r, n_kv, d, dtype=dtype)
    proj.set_kv(0, wk, wv); ad.set_a(0, a)
    for i in range(A):
        ad.set_b(0, i, b[i], 16.0)
    pool.append_tokens(L)
    agents = range(A) if scheme == "NonShared" else [1]
    for i in agents:
        assert pool.append_kv_project(proj, 0, i, 0, x, merge=ad) == L
        want_k = orc.apply_rope(orc.matmul(x, wk), n_kv, d, 0)
        want_v = orc.matmul(x, wv) + np.float32(16.0 / r) * orc.matmul(orc.matmul(x, a), b[i])
        got_k, got_v = pool.key_view(0, i), pool.value_view(0, i)
        if bf16:
            assert ctx.last_kernel() == "kv_project_umma"
            assert orc.max_rel_error(got_k, want_k) <= 4e-3 and orc.max_rel_error(got_v, want_v) <= 4e-3
        else:
            assert np.array_equal(got_v, want_v)                     # the reference's order, bit for bit
            assert orc.max_rel_error(got_k, want_k) <= 1e-6
    if scheme == "FullShared":                                       # the next agent finds the rows there (first writer wins)
        assert pool.append_kv_project(proj, 0, 0, 0, x, merge=ad) == 0
    pool.close(); proj.close(); ad.close()


@pytest.mark.parametrize("n_rows", [1, 3, 8])
def test_decode_step_rows_take_the_gemv_path(ctx, orc, n_rows):
    """<= 8 new rows (a decode step) stream the packed weights as GEMVs over all SMs (rows_project.cu) instead of one
    128-row tcgen05 tile: K / V (+ value adapter), V_lr and q must equal what the GEMM path gives for the same rows."""
    from paper_2602_01053_b200 import Adapters, Pool, Projection, abi
    L0, d_model, n_q, n_kv, d, r, A = 45, 256, 8, 2, 128, 16, 2
    L = L0 + n_rows
    x, wk, wv = make_inputs(orc, 6100 + n_rows, L, d_model, n_kv, d, True)
    rnd = orc.round_bf16
    wq = rnd(orc.gaussian(d_model, n_q * d, orc.child(61, 2), 1.0 / np.sqrt(d_model), np.float32))
    a = rnd(orc.gaussian(d_model, r, orc.child(61, 3), 1.0 / np.sqrt(d_model), np.float32))
    bq = [rnd(orc.gaussian(r, n_q * d, orc.child(61, 10 + i), 0.02 / np.sqrt(r), np.float32)) for i in range(A)]
    bv = [rnd(orc.gaussian(r, n_kv * d, orc.child(61, 20 + i), 0.02 / np.sqrt(r), np.float32)) for i in range(A)]
    for scheme, merge in (("BaseLRShared", False), ("FullShared", True)):
        pool = Pool(ctx, scheme, 1, n_kv, d, d_model, 0 if merge else r, A, max_tokens=L, dtype=abi.BF16, page_tokens=16)
        proj = Projection(ctx, 1, d_model, n_kv, d, dtype=abi.BF16)
        ad = Adapters(ctx, 1, A, d_model, r, n_kv, d, dtype=abi.BF16)
        proj.set_kv(0, wk, wv); proj.set_q(0, n_q, wq); ad.set_a(0, a)
        for i in range(A):
            proj.set_q_lora(0, i, A, a, bq[i], 16.0); ad.set_b(0, i, bv[i], 16.0)
        pool.append_tokens(L)
        kw = dict(merge=ad) if merge else {}
        assert pool.append_kv_project(proj, 0, 1, 0, x[:L0], **kw) == L0          # the GEMM path
        assert ctx.last_kernel() == "kv_project_umma"
        assert pool.append_kv_project(proj, 0, 1, L0, x[L0:], **kw) == n_rows     # the GEMV path, mid-page
        assert ctx.last_kernel() == "rows_kv_project"
        want_k = orc.apply_rope(orc.matmul(x, wk), n_kv, d, 0)
        want_v = orc.matmul(x, wv) + (np.float32(16.0 / r) * orc.matmul(orc.matmul(x, a), bv[1]) if merge else 0)
        assert orc.max_rel_error(pool.key_view(0, 1 if scheme == "NonShared" else 0), want_k) <= 4e-3
        assert orc.max_rel_error(pool.value_view(0, 0), want_v) <= 4e-3
        if not merge:
            assert pool.append_lr_project(ad, 0, 0, 0, x[:L0]) == L0
            assert pool.append_lr_project(ad, 0, 0, L0, x[L0:]) == n_rows
            assert orc.max_rel_error(pool.lr_view(0, 0), orc.matmul(x, a)) <= 4e-3
        got_q = proj.query(0, 1, L0, x[L0:], n_q * d)
        assert ctx.last_kernel() == "rows_q_project"
        want_q = reference_q(orc, x[L0:], wq, a, bq[1], 16.0, n_q, d, L0, True)
        assert orc.max_rel_error(got_q, want_q) <= 1e-4
        assert orc.max_rel_error(proj.query(0, -1, L0, x[L0:], n_q * d), reference_q(orc, x[L0:], wq, None, None, 16.0, n_q, d, L0, True)) <= 1e-4
        pool.close(); proj.close(); ad.close()


@pytest.mark.parametrize("L,d_model,n_q,n_kv,r,chunks,shard", [
    (600, 256, 8, 2, 16, (600,), None),
    (1000, 512, 16, 4, 64, (300, 700), (2, 2)),      # second chunk starts mid-page; this shard holds kv heads 2..3
    (420, 4096, 4, 2, 8, (420,), None),              # the Llama reduction depth: 6 x 4096 / 16 accumulate steps
])
def test_fp32_projections_on_the_tensor_cores_stay_at_fp32_accuracy(ctx, orc, L, d_model, n_q, n_kv, r, chunks, shard):
    """fp32 pools with >= 256 rows per call: x Wk / x Wv / x Wq run on the tcgen05 GEMM over bf16 planes of the fp32 operands
    (six plane products along K, kv_project_umma.cu), the adapter terms as fp32 FMAs in the epilogue.  fp32-accurate (<= 1e-5
    here; the north star's fp32 mode asks 1e-4), not the reference's summation order -- kernel policy 2 keeps that."""
    from paper_2602_01053_b200 import Adapters, Pool, Projection, abi
    d, A = 128, 2
    x, wk, wv = make_inputs(orc, 7700 + L, L, d_model, n_kv, d, False)
    wq = orc.gaussian(d_model, n_q * d, orc.child(L, 2), 1.0 / np.sqrt(d_model), np.float32)
    a = orc.gaussian(d_model, r, orc.child(L, 3), 1.0 / np.sqrt(d_model), np.float32)
    bq = [orc.gaussian(r, n_q * d, orc.child(L, 10 + i), 0.3 / np.sqrt(r), np.float32) for i in range(A)]
    bv = [orc.gaussian(r, n_kv * d, orc.child(L, 20 + i), 0.3 / np.sqrt(r), np.float32) for i in range(A)]
    kb, kn = shard if shard else (0, n_kv)
    g = n_q // n_kv
    kv_cols, q_cols = slice(kb * d, (kb + kn) * d), slice(kb * g * d, (kb + kn) * g * d)
    want_k, want_v = reference_kv(orc, x, wk, wv, n_kv, d, 0, True)
    for scheme, merge in (("BaseLRShared", False), ("FullShared", True)):
        pool = Pool(ctx, scheme, 1, n_kv, d, d_model, 0 if merge else r, A, max_tokens=L, dtype=abi.F32, page_tokens=64,
                    kv_head_begin=kb, n_kv_local=kn)
        proj = Projection(ctx, 1, d_model, n_kv, d, kv_head_begin=kb, n_kv_local=kn, dtype=abi.F32)
        ad = Adapters(ctx, 1, A, d_model, r, n_kv, d, dtype=abi.F32, kv_head_begin=kb, n_kv_local=kn)
        proj.set_kv(0, wk, wv); ad.set_a(0, a)
        for i in range(A):
            ad.set_b(0, i, bv[i], 16.0)
        pool.append_tokens(L)
        row = 0
        for n in chunks:
            assert pool.append_kv_project(proj, 0, 1, row, x[row:row + n], merge=ad if merge else None) == n
            assert ctx.last_kernel() == "kv_project_planes"
            row += n
        wv_full = want_v + (np.float32(16.0 / r) * orc.matmul(orc.matmul(x, a), bv[1]) if merge else 0)
        assert orc.max_rel_error(pool.key_view(0, 1), want_k[:, kv_cols]) <= 1e-5
        assert orc.max_rel_error(pool.value_view(0, 1), wv_full[:, kv_cols]) <= 1e-5
        pool.close(); proj.close(); ad.close()
    # the query side, with the q adapter and the rotation at an offset position
    proj = Projection(ctx, 1, d_model, n_kv, d, kv_head_begin=kb, n_kv_local=kn, dtype=abi.F32)
    proj.set_q(0, n_q, wq)
    for i in range(A):
        proj.set_q_lora(0, i, A, a, bq[i], 16.0)
    for agent in (1, -1):
        got = proj.query(0, agent, 77, x, kn * g * d, rope=True)
        assert ctx.last_kernel() == "q_project_planes"
        want = reference_q(orc, x, wq, a if agent >= 0 else None, bq[agent] if agent >= 0 else None, 16.0, n_q, d, 77, True)[:, q_cols]
        assert orc.max_rel_error(got, want) <= 1e-5, agent
    ctx.set_kernel_policy(2)            # the reference's summation order, bit for bit without the rotation
    try:
        got = proj.query(0, 1, 77, x, kn * g * d, rope=False)
        assert ctx.last_kernel() == "q_project_f32"
        assert np.array_equal(got, reference_q(orc, x, wq, a, bq[1], 16.0, n_q, d, 77, False)[:, q_cols])
    finally:
        ctx.set_kernel_policy(0)
    proj.close()
