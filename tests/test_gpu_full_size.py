"""BASELINE-size checks through size-independent properties (the CPU oracle needs ~1 s per head at this size, so
only a sample of heads is compared directly; bench.py compares a whole layer in every run).  One layer of cfg 2:
Llama-3.1-8B attention shape (32 q / 8 kv heads, d = 128), rank 16, 3 agents, 32 768 cached tokens, bf16 pages.
Needs a B200."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

N_Q, N_KV, D, R, A, L, D_MODEL = 32, 8, 128, 16, 3, 32768, 256


@pytest.fixture(scope="module")
def ctx():
    from paper_2602_01053_b200 import Context
    c = Context(0)
    yield c
    c.close()


@pytest.fixture(scope="module")
def layer(orc):
    rnd = orc.round_bf16
    g = lambda rows, cols, key, scale: rnd(orc.gaussian(rows, cols, orc.child(2602, key), scale, np.float32))
    return dict(k=g(L, N_KV * D, 2, 1.0 / np.sqrt(D)), v=g(L, N_KV * D, 3, 1.0), v2=g(L, N_KV * D, 13, 1.0),
                lr=g(L, R, 4, 1.0), lr2=g(L, R, 14, 1.0),
                b=[g(R, N_KV * D, 20 + a, 0.02 / np.sqrt(R)) for a in range(A)],
                q=np.stack([g(1, N_Q * D, 30 + a, 1.0 / np.sqrt(D))[0] for a in range(A)]))


def build(ctx, layer, v, lr, kv_begin=0, n_kv_local=0, page_tokens=0):
    from paper_2602_01053_b200 import Adapters, Pool, abi
    pool = Pool(ctx, "BaseLRShared", 1, N_KV, D, D_MODEL, R, A, max_tokens=L, dtype=abi.BF16, page_tokens=page_tokens,
                kv_head_begin=kv_begin, n_kv_local=n_kv_local)
    ad = Adapters(ctx, 1, A, D_MODEL, R, N_KV, D, kv_head_begin=kv_begin, n_kv_local=n_kv_local, dtype=abi.BF16)
    pool.append_tokens(L)
    pool.append_key(0, 0, 0, layer["k"]); pool.append_value(0, 0, 0, v); pool.append_lr(0, 0, 0, lr)
    for a in range(A):
        ad.set_b(0, a, layer["b"][a], 16.0)
    return pool, ad


def decode(pool, ad, q):
    return pool.decode(ad, 0, 1, list(range(A)), N_Q, q[None])[0]


def test_full_size_decode_properties(ctx, orc, layer):
    g = N_Q // N_KV
    pool, ad = build(ctx, layer, layer["v"], layer["lr"])
    out = decode(pool, ad, layer["q"])
    assert ctx.last_kernel() == "fla_decode_tma"
    # (1) a sample of heads against the reference path (gqa_attention per agent, attention.hpp:332-363)
    for a, kvh in ((0, 0), (2, 5)):
        cols = slice(kvh * D, (kvh + 1) * D)
        qh = layer["q"][a][None, kvh * g * D:(kvh + 1) * g * D]
        want = orc.gqa_attention(np.ascontiguousarray(qh), np.ascontiguousarray(layer["k"][:, cols]),
                                 np.ascontiguousarray(layer["v"][:, cols]), layer["lr"], np.ascontiguousarray(layer["b"][a][:, cols]),
                                 16.0 / R, L - 1, g, 1)
        assert orc.max_rel_error(out[a][None, kvh * g * D:(kvh + 1) * g * D], want) <= 2e-2
    # (2) kv-head shards (no communication inside attention) give the shard's slice of the output.  The stream-K split
    # points depend on how many heads a GPU holds and every split rounds P to bf16 against its own running maximum, so
    # the two partitions differ by bf16-P rounding noise (the same size as the distance to the fp32 oracle), not more
    for kb, kn in ((0, 4), (6, 2), (3, 1)):
        sp, sa = build(ctx, layer, layer["v"], layer["lr"], kv_begin=kb, n_kv_local=kn)
        q_local = np.ascontiguousarray(layer["q"][:, kb * g * D:(kb + kn) * g * D])
        got = sp.decode(sa, 0, 1, list(range(A)), N_Q, q_local[None])[0]
        assert orc.max_rel_error(got, out[:, kb * g * D:(kb + kn) * g * D]) <= 5e-3, (kb, kn)
        sp.close(); sa.close()
    # (3) the page size is a layout choice: another one gives the same numbers up to the split-merge order
    p2, a2 = build(ctx, layer, layer["v"], layer["lr"], page_tokens=256)
    assert orc.max_rel_error(decode(p2, a2, layer["q"]), out) <= 5e-3
    p2.close(); a2.close()
    # (4) the CUDA-core kernels (policy 1) agree with the tensor-core path far inside the oracle tolerance
    ctx.set_kernel_policy(1)
    ref = decode(pool, ad, layer["q"])
    ctx.set_kernel_policy(0)
    assert ctx.last_kernel() == "fla_paged_simt"
    assert orc.max_rel_error(out, ref) <= 5e-3
    # (5) linearity in the values: the same q, K (hence the same softmax weights) over V + V2 and V_lr + V_lr2
    pb, ab = build(ctx, layer, layer["v2"], layer["lr2"])
    out2 = decode(pb, ab, layer["q"])
    pb.close(); ab.close()
    vs, ls = orc.round_bf16(layer["v"] + layer["v2"]), orc.round_bf16(layer["lr"] + layer["lr2"])
    exact = np.array_equal(vs, layer["v"] + layer["v2"]) and np.array_equal(ls, layer["lr"] + layer["lr2"])
    pc, ac = build(ctx, layer, vs, ls)
    out12 = decode(pc, ac, layer["q"])
    pc.close(); ac.close()
    # the sums are re-rounded to bf16 (half an ulp per element, averaged over 32K keys), hence the looser bound
    assert orc.max_rel_error(out12, out + out2) <= (1e-4 if exact else 3e-3)
    pool.close(); ad.close()


def test_full_size_prefill_block_against_decode(ctx, orc, layer):
    """The last row of a prefill block at query_offset = L - L_c sees the whole cache: it must equal the decode
    output of the same query (two different kernels, tcgen05 prefill vs. the streaming decode kernel)."""
    pool, ad = build(ctx, layer, layer["v"], layer["lr"])
    L_c = 64
    q = orc.round_bf16(orc.gaussian(L_c, N_Q * D, 777, 1.0 / np.sqrt(D), np.float32))
    blk = pool.prefill(ad, 0, 1, N_Q, q, L - L_c)
    assert ctx.last_kernel() == "fla_prefill_umma"
    one = pool.decode(ad, 0, 1, [1], N_Q, q[None, L_c - 1:L_c])[0]
    assert orc.max_rel_error(blk[L_c - 1:L_c], one) <= 2e-3
    pool.close(); ad.close()


def test_full_size_projections_sampled_rows(ctx, orc):
    """cfg 3's append: 16 384 new rows x d_model 4096 through the persistent tcgen05 projection kernels (2 048 tiles over 148
    CTAs, every CTA walks ~14 tiles) -- a seeded sample of rows against matmul / apply_rope / the LoRA terms of the
    reference path (engine.hpp:362-403), K / V / V_lr read back from the pages, q from the query projection."""
    import torch
    from paper_2602_01053_b200 import Adapters, Pool, Projection, abi
    n_rows, d_model, r, row0 = 16384, 4096, R, 0
    dev = torch.device("cuda", 0)
    gen = torch.Generator(device=dev); gen.manual_seed(5)
    x_dev = torch.randn((n_rows, d_model), generator=gen, device=dev, dtype=torch.float32).to(torch.bfloat16).to(torch.float32)
    rnd = orc.round_bf16
    g = lambda rows, cols, key, scale: rnd(orc.gaussian(rows, cols, orc.child(303, key), scale, np.float32))
    wq, wk, wv = g(d_model, N_Q * D, 1, d_model ** -0.5), g(d_model, N_KV * D, 2, d_model ** -0.5), g(d_model, N_KV * D, 3, d_model ** -0.5)
    a_q, a_v = g(d_model, r, 4, d_model ** -0.5), g(d_model, r, 5, d_model ** -0.5)
    b_q = g(r, N_Q * D, 6, 0.02 / np.sqrt(r))
    pool = Pool(ctx, "BaseLRShared", 1, N_KV, D, d_model, r, 1, max_tokens=n_rows, dtype=abi.BF16)
    proj = Projection(ctx, 1, d_model, N_KV, D, dtype=abi.BF16)
    ad = Adapters(ctx, 1, 1, d_model, r, N_KV, D, dtype=abi.BF16)
    proj.set_kv(0, wk, wv); proj.set_q(0, N_Q, wq); proj.set_q_lora(0, 0, 1, a_q, b_q, 16.0); ad.set_a(0, a_v)
    pool.append_tokens(n_rows)
    torch.cuda.synchronize()
    assert pool.append_kv_project(proj, 0, 0, row0, dev_ptr=x_dev.data_ptr(), n_rows=n_rows, ld=d_model) == n_rows
    assert ctx.last_kernel() == "kv_project_umma"
    assert pool.append_lr_project(ad, 0, 0, row0, dev_ptr=x_dev.data_ptr(), n_rows=n_rows, ld=d_model) == n_rows
    q_dev = torch.empty((n_rows, N_Q * D), device=dev, dtype=torch.float32)
    proj.query_device(0, 0, row0, x_dev.data_ptr(), n_rows, d_model, q_dev.data_ptr())
    assert ctx.last_kernel() == "q_project_umma"
    ctx.synchronize()
    rows = np.array([0, 1, 127, 128, 5000, 9999, 16255, 16383])      # first / last tiles, tile edges, the middle
    xs = x_dev[torch.from_numpy(rows).to(dev)].cpu().numpy()
    k_got, v_got, lr_got = pool.key_view(0, 0)[rows], pool.value_view(0, 0)[rows], pool.lr_view(0, 0)[rows]
    q_got = q_dev[torch.from_numpy(rows).to(dev)].cpu().numpy()
    for i, row in enumerate(rows):
        xi = xs[i:i + 1]
        k_want = orc.apply_rope(orc.matmul(xi, wk), N_KV, D, int(row))
        q_want = orc.apply_rope(orc.matmul(xi, wq) + np.float32(16.0 / r) * orc.matmul(orc.matmul(xi, a_q), b_q), N_Q, D, int(row))
        assert orc.max_rel_error(k_got[i:i + 1], k_want) <= 4e-3, row
        assert orc.max_rel_error(v_got[i:i + 1], orc.matmul(xi, wv)) <= 4e-3, row
        assert orc.max_rel_error(lr_got[i:i + 1], orc.matmul(xi, a_v)) <= 4e-3, row
        assert orc.max_rel_error(q_got[i:i + 1], q_want) <= 1e-4, row
    pool.close(); proj.close(); ad.close()
