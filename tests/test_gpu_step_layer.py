"""lorakv_step_layer: one decode layer-step of step() on the attention sublayer (proj/include/lorakv/engine.hpp:331-443) --
projections of the new rows (q with q-LoRA and RoPE, K with RoPE, V [+ merged value adapter]), the appends (K, V, V_lr = x A_v)
and Flash-LoRA-Attention over the store -- as four chained launches (csrc/step_layer.cu + the decode kernels).

Checked against (a) the same step composed from the reference path on the CPU (checker: matmul, apply_rope, gqa_attention)
and (b) the separate C-ABI entry points it replaces (append_kv_project[_full], append_lr_project, proj_query, fla_prefill),
for every scheme of the hot path, 1...8 rows, kv-head shards and a generation loop that crosses page boundaries."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    import paper_2602_01053_b200 as pkg
    c = pkg.Context(0)
    yield c
    c.close()


def weights(orc, seed, d_model, n_q, n_kv, d, r, A):
    rnd = orc.round_bf16
    g = lambda rows, cols, key, scale: rnd(orc.gaussian(rows, cols, orc.child(seed, key), scale, np.float32))
    s = 1.0 / np.sqrt(d_model)
    return dict(wq=g(d_model, n_q * d, 1, s), wk=g(d_model, n_kv * d, 2, s), wv=g(d_model, n_kv * d, 3, s),
                a_q=g(d_model, r, 4, s), a_v=[g(d_model, r, 40 + i, s) for i in range(A)],
                b_q=[g(r, n_q * d, 10 + i, 0.02 / np.sqrt(r)) for i in range(A)],
                b_v=[g(r, n_kv * d, 20 + i, 0.02 / np.sqrt(r)) for i in range(A)])


def build(ctx, scheme, w, d_model, n_q, n_kv, d, r, A, L, P, shard=(0, 0)):
    from paper_2602_01053_b200 import Adapters, Pool, Projection, abi
    full = scheme in ("NonShared", "FullShared")
    kb, kl = shard
    pool = Pool(ctx, scheme, 1, n_kv, d, d_model, 0 if full else r, A, max_tokens=L, dtype=abi.BF16, page_tokens=P,
                kv_head_begin=kb, n_kv_local=kl)
    proj = Projection(ctx, 1, d_model, n_kv, d, kv_head_begin=kb, n_kv_local=kl, dtype=abi.BF16)
    ad = Adapters(ctx, 1, A, d_model, r, n_kv, d, kv_head_begin=kb, n_kv_local=kl, dtype=abi.BF16)
    proj.set_kv(0, w["wk"], w["wv"]); proj.set_q(0, n_q, w["wq"])
    per_agent_a = scheme == "BaseShared"
    if not per_agent_a:
        ad.set_a(0, w["a_v"][0])
    for i in range(A):
        proj.set_q_lora(0, i, A, w["a_q"], w["b_q"][i], 16.0)
        if per_agent_a:
            ad.set_a_agent(0, i, w["a_v"][i])
        ad.set_b(0, i, w["b_v"][i], 16.0)
    return pool, proj, ad


def reference_step(orc, scheme, w, x, rows, agent, n_q, n_kv, d, r):
    """q rows and attention output of rows [rows[0], rows[1]) over the whole trajectory x[:rows[1]], composed from the reference path."""
    full = scheme in ("NonShared", "FullShared")
    a_v = w["a_v"][agent] if scheme == "BaseShared" else w["a_v"][0]
    s = np.float32(16.0 / r)
    p0, p1 = rows
    xs = x[:p1]
    k = orc.apply_rope(orc.matmul(xs, w["wk"]), n_kv, d, 0)
    v = orc.matmul(xs, w["wv"])
    if full:
        v = v + s * orc.matmul(orc.matmul(xs, a_v), w["b_v"][agent])
    q = orc.matmul(x[p0:p1], w["wq"]) + s * orc.matmul(orc.matmul(x[p0:p1], w["a_q"]), w["b_q"][agent])
    q = orc.apply_rope(q, n_q, d, p0)
    if full:
        out = orc.gqa_attention(q, k, v, np.zeros((p1, 0), np.float32), np.zeros((0, n_kv * d), np.float32), 1.0, p0, n_q, n_kv)
    else:
        out = orc.gqa_attention(q, k, v, orc.matmul(xs, a_v), w["b_v"][agent], float(s), p0, n_q, n_kv)
    return q, out


@pytest.mark.parametrize("scheme", ["BaseLRShared", "BaseShared", "FullShared", "NonShared"])
@pytest.mark.parametrize("n_rows", [1, 2, 8])
def test_step_layer_matches_the_reference_step(ctx, orc, scheme, n_rows):
    import torch
    d_model, n_q, n_kv, d, r, A, P = 256, 8, 2, 128, 16, 2, 16
    L0, agent = 37, 1
    L = L0 + n_rows
    w = weights(orc, 7300 + n_rows, d_model, n_q, n_kv, d, r, A)
    x = orc.round_bf16(orc.gaussian(L, d_model, orc.child(7301, n_rows), 1.0, np.float32))
    full = scheme in ("NonShared", "FullShared")
    pool, proj, ad = build(ctx, scheme, w, d_model, n_q, n_kv, d, r, A, L, P)
    pool.append_tokens(L)
    # context rows through the separate entry points (the prefill path)
    if full:
        assert pool.append_kv_project(proj, 0, agent, 0, x[:L0], merge=ad) == L0
    else:
        assert pool.append_kv_project(proj, 0, agent, 0, x[:L0]) == L0
        assert pool.append_lr_project(ad, 0, agent, 0, x[:L0]) == L0
    launches0 = ctx.launch_count
    xd = torch.from_numpy(x[L0:]).cuda()
    qd = torch.zeros((n_rows, n_q * d), device="cuda"); od = torch.zeros_like(qd)
    torch.cuda.synchronize()
    pool.step_layer_device(proj, ad, 0, agent, L0, xd.data_ptr(), n_rows, d_model, n_q, od.data_ptr(), q_dev=qd.data_ptr())
    ctx.synchronize()
    if n_rows == 1:
        assert ctx.launch_count - launches0 == 4                   # projections (2), attention, merge epilogue
        assert ctx.last_kernel() == "fla_decode_tma"
    want_q, want = reference_step(orc, scheme, w, x, (L0, L), agent, n_q, n_kv, d, r)
    assert orc.max_rel_error(qd.cpu().numpy(), want_q) <= 1e-4
    assert orc.max_rel_error(od.cpu().numpy(), want) <= 2e-2
    # the caches hold what the separate entry points would have stored
    set_agent = agent
    assert pool.rows(0, 0, set_agent) == L and pool.rows(1, 0, set_agent) == L
    k_all = orc.apply_rope(orc.matmul(x, w["wk"]), n_kv, d, 0)
    assert orc.max_rel_error(pool.key_view(0, set_agent), k_all) <= 4e-3
    if not full:
        a_v = w["a_v"][agent] if scheme == "BaseShared" else w["a_v"][0]
        assert pool.rows(2, 0, set_agent) == L
        assert orc.max_rel_error(pool.lr_view(0, set_agent), orc.matmul(x, a_v)) <= 4e-3
    pool.close(); proj.close(); ad.close()


def test_step_layer_equals_the_separate_entry_points(ctx, orc):
    """Same rows through lorakv_step_layer (fused, DEVICE) and through the four calls it replaces (HOST): identical cache
    rows bit for bit (same kernels' arithmetic order is not required -- bf16 pages round both to the same values or one ulp),
    attention outputs within the bf16 tolerance; and a HOST call of step_layer takes the generic route and agrees too."""
    import torch
    d_model, n_q, n_kv, d, r, A, P = 512, 16, 4, 128, 16, 3, 32
    L0, n_gen = 60, 9                                              # the generation crosses a page boundary at row 64
    w = weights(orc, 8100, d_model, n_q, n_kv, d, r, A)
    x = orc.round_bf16(orc.gaussian(L0 + n_gen, d_model, orc.child(8101, 1), 1.0, np.float32))
    outs = {}
    for mode in ("fused", "separate", "host"):
        pool, proj, ad = build(ctx, "BaseLRShared", w, d_model, n_q, n_kv, d, r, A, L0 + n_gen, P)
        pool.append_tokens(L0)
        pool.append_kv_project(proj, 0, 0, 0, x[:L0]); pool.append_lr_project(ad, 0, 0, 0, x[:L0])
        got = []
        for t in range(n_gen):
            agent, row = t % A, L0 + t
            pool.append_tokens(1)
            if mode == "fused":
                xd = torch.from_numpy(x[row:row + 1]).cuda(); od = torch.zeros((1, n_q * d), device="cuda")
                pool.step_layer_device(proj, ad, 0, agent, row, xd.data_ptr(), 1, d_model, n_q, od.data_ptr())
                ctx.synchronize()
                assert ctx.last_kernel() == "fla_decode_tma"
                got.append(od.cpu().numpy())
            elif mode == "host":
                got.append(pool.step_layer(proj, ad, 0, agent, row, x[row:row + 1], n_q)[1])
            else:
                pool.append_kv_project(proj, 0, agent, row, x[row:row + 1]); pool.append_lr_project(ad, 0, agent, row, x[row:row + 1])
                q = proj.query(0, agent, row, x[row:row + 1], n_q * d)
                got.append(pool.prefill(ad, 0, agent, n_q, q, row))
        outs[mode] = (np.concatenate(got), pool.key_view(0, 0), pool.value_view(0, 0), pool.lr_view(0, 0), pool.page_table())
        pool.close(); proj.close(); ad.close()
    for mode in ("fused", "host"):
        o, k, v, lr, pt = outs[mode]
        o2, k2, v2, lr2, pt2 = outs["separate"]
        assert np.array_equal(pt, pt2)                              # page tables bit-exact
        assert orc.max_rel_error(k, k2) <= 4e-3 and orc.max_rel_error(v, v2) <= 4e-3 and orc.max_rel_error(lr, lr2) <= 4e-3
        assert orc.max_rel_error(o, o2) <= 2e-2
    # and the whole generation against the reference path
    for t in range(n_gen):
        _q, want = reference_step(orc, "BaseLRShared", w, x, (L0 + t, L0 + t + 1), t % A, n_q, n_kv, d, r)
        assert orc.max_rel_error(outs["fused"][0][t:t + 1], want) <= 2e-2


def test_step_layer_generation_soak(ctx, orc):
    """150 tokens x 3 layers through the dependent-launch chain without a host synchronisation in between (the prefetch before
    the wait sees a pending page write on every call; pages fill up and new ones are allocated 4 times): the caches must end
    up equal to what the separate entry points store, the last token's outputs equal the reference path."""
    import torch
    d_model, n_q, n_kv, d, r, A, P, n_layers = 256, 8, 2, 128, 16, 3, 32, 3
    L0, n_gen = 10, 150
    ws = [weights(orc, 8400 + l, d_model, n_q, n_kv, d, r, A) for l in range(n_layers)]
    x = orc.round_bf16(orc.gaussian(L0 + n_gen, d_model, orc.child(8401, 1), 1.0, np.float32))
    from paper_2602_01053_b200 import Adapters, Pool, Projection, abi
    pool = Pool(ctx, "BaseLRShared", n_layers, n_kv, d, d_model, r, A, max_tokens=L0 + n_gen, dtype=abi.BF16, page_tokens=P)
    proj = Projection(ctx, n_layers, d_model, n_kv, d, dtype=abi.BF16)
    ad = Adapters(ctx, n_layers, A, d_model, r, n_kv, d, dtype=abi.BF16)
    for l, w in enumerate(ws):
        proj.set_kv(l, w["wk"], w["wv"]); proj.set_q(l, n_q, w["wq"]); ad.set_a(l, w["a_v"][0])
        for i in range(A):
            proj.set_q_lora(l, i, A, w["a_q"], w["b_q"][i], 16.0); ad.set_b(l, i, w["b_v"][i], 16.0)
    pool.append_tokens(L0)
    for l in range(n_layers):
        pool.append_kv_project(proj, l, 0, 0, x[:L0]); pool.append_lr_project(ad, l, 0, 0, x[:L0])
    xd = torch.from_numpy(x).cuda()
    od = torch.zeros((n_gen, n_layers, n_q * d), device="cuda")
    for t in range(n_gen):
        pool.append_tokens(1)
        for l in range(n_layers):
            pool.step_layer_device(proj, ad, l, t % A, L0 + t, xd[L0 + t].data_ptr(), 1, d_model, n_q, od[t, l].data_ptr())
    ctx.synchronize()
    got = od.cpu().numpy()
    for l, w in enumerate(ws):
        assert pool.rows(0, l, 0) == L0 + n_gen and pool.rows(2, l, 0) == L0 + n_gen
        assert orc.max_rel_error(pool.key_view(l, 0), orc.apply_rope(orc.matmul(x, w["wk"]), n_kv, d, 0)) <= 4e-3
        assert orc.max_rel_error(pool.value_view(l, 0), orc.matmul(x, w["wv"])) <= 4e-3
        assert orc.max_rel_error(pool.lr_view(l, 0), orc.matmul(x, w["a_v"][0])) <= 4e-3
        for t in (0, 21, 22, 53, 54, n_gen - 1):          # around the page boundaries (rows 32, 64) and the ends
            _q, want = reference_step(orc, "BaseLRShared", w, x, (L0 + t, L0 + t + 1), t % A, n_q, n_kv, d, r)
            assert orc.max_rel_error(got[t, l][None, :], want) <= 2e-2, (l, t)
    pool.close(); proj.close(); ad.close()


def test_step_layer_on_a_kv_head_shard(ctx, orc):
    """A rank holding kv heads [1, 3) of 4: its q / output columns are the matching slice of the single-GPU step."""
    import torch
    d_model, n_q, n_kv, d, r, A, P = 256, 8, 4, 128, 16, 2, 16
    L0 = 20
    w = weights(orc, 8200, d_model, n_q, n_kv, d, r, A)
    x = orc.round_bf16(orc.gaussian(L0 + 1, d_model, orc.child(8201, 1), 1.0, np.float32))
    g = n_q // n_kv
    pool, proj, ad = build(ctx, "BaseLRShared", w, d_model, n_q, n_kv, d, r, A, L0 + 1, P, shard=(1, 2))
    pool.append_tokens(L0 + 1)
    pool.append_kv_project(proj, 0, 0, 0, x[:L0]); pool.append_lr_project(ad, 0, 0, 0, x[:L0])
    xd = torch.from_numpy(x[L0:]).cuda()
    qd = torch.zeros((1, 2 * g * d), device="cuda"); od = torch.zeros_like(qd)
    pool.step_layer_device(proj, ad, 0, 1, L0, xd.data_ptr(), 1, d_model, n_q, od.data_ptr(), q_dev=qd.data_ptr())
    ctx.synchronize()
    want_q, want = reference_step(orc, "BaseLRShared", w, x, (L0, L0 + 1), 1, n_q, n_kv, d, r)
    cols = slice(1 * g * d, 3 * g * d)
    assert orc.max_rel_error(qd.cpu().numpy(), want_q[:, cols]) <= 1e-4
    assert orc.max_rel_error(od.cpu().numpy(), want[:, cols]) <= 2e-2
    pool.close(); proj.close(); ad.close()


def test_step_layer_errors(ctx, orc):
    from paper_2602_01053_b200 import abi
    d_model, n_q, n_kv, d, r, A, P = 256, 8, 2, 128, 16, 2, 16
    w = weights(orc, 8300, d_model, n_q, n_kv, d, r, A)
    x = orc.round_bf16(orc.gaussian(4, d_model, orc.child(8301, 1), 1.0, np.float32))
    pool, proj, ad = build(ctx, "BaseLRShared", w, d_model, n_q, n_kv, d, r, A, 64, P)
    pool.append_tokens(8)
    with pytest.raises(abi.LorakvError, match="gap"):               # rows must continue the cache (kvcache.hpp:400-407)
        pool.step_layer(proj, ad, 0, 0, 3, x[:1], n_q)
    with pytest.raises(abi.LorakvError, match="no adapter tables"):
        pool.step_layer(proj, None, 0, 0, 0, x[:1], n_q)
    with pytest.raises(abi.LorakvError, match="unknown agent"):
        pool.step_layer(proj, ad, 0, 5, 0, x[:1], n_q)
    pool.close(); proj.close(); ad.close()
