import numpy as np, sys
sys.path.insert(0, "/root/repo")
from oracle import checker
import paper_2602_01053_b200 as pkg
from paper_2602_01053_b200 import abi
from tests.test_gpu_pool import build_pool
orc = checker.oracle()
ctx = pkg.Context(0)
import os
F32_ONLY = os.environ.get("LORAKV_SMOKE_F32_ONLY") == "1"    # synccheck: only the mbarrier rings of the fp32 kernels and the gather
# decode MW=1 and MW=2/KT=2, prefill umma, lr_project, selftest
for (n_q, n_kv, d, r, A, L, P) in ([] if F32_ONLY else [(8, 2, 128, 16, 3, 200, 64), (8, 2, 128, 32, 8, 150, 32), (16, 2, 64, 8, 12, 100, 16)]):
    pool, ad, layers = build_pool(ctx, orc, "BaseLRShared", abi.BF16, 7, L, 1, n_q, n_kv, d, r, A, P=P, project=True, d_model=192)
    q, k, v, v_lr, b, s = layers[0]
    out = pool.decode(ad, 0, 1, list(range(A)), n_q, np.stack([q[a][0] for a in range(A)])[None])
    want = orc.gqa_attention(q[1], k, v, v_lr, b[1], s, L - 1, n_q, n_kv)
    print("decode", ctx.last_kernel(), orc.max_rel_error(out[0, 1][None, :], want))
    qp = orc.round_bf16(orc.gaussian(40, n_q * d, 5, 1.0 / np.sqrt(d), np.float32))
    got = pool.prefill(ad, 0, 1, n_q, qp, L - 40)
    want = orc.gqa_attention(qp, k, v, v_lr, b[1], s, L - 40, n_q, n_kv)
    print("prefill", ctx.last_kernel(), orc.max_rel_error(got, want))
    pool.close()
# fp32 mode: split-TF32 decode (one- and two-warp workers) and prefill over chunk-swizzled fp32 pages; the peer-memory
# output gather with one rank (merge epilogue storing into the gather buffer + handshake kernel)
from paper_2602_01053_b200 import Gather
for (n_q, n_kv, d, r, A, L, P) in [(8, 2, 128, 16, 3, 203, 64), (8, 2, 64, 32, 8, 150, 8)]:
    pool, ad, layers = build_pool(ctx, orc, "BaseLRShared", abi.F32, 9, L, 1, n_q, n_kv, d, r, A, P=P)
    q, k, v, v_lr, b, s = layers[0]
    qs = np.stack([q[a][0] for a in range(A)])[None]
    out = pool.decode(ad, 0, 1, list(range(A)), n_q, qs)
    want = orc.gqa_attention(q[1], k, v, v_lr, b[1], s, L - 1, n_q, n_kv)
    print("decode", ctx.last_kernel(), orc.max_rel_error(out[0, 1][None, :], want))
    gth = Gather(ctx, 0, 1, qs.size)
    for _ in range(2):
        full, _dev = pool.decode_gather(ad, gth, 0, 1, list(range(A)), n_q, q=qs)
    print("gather", ctx.last_kernel(), bool(np.array_equal(full, out)))
    gth.close()
    qp = orc.gaussian(40, n_q * d, 5, 1.0 / np.sqrt(d), np.float32)
    got = pool.prefill(ad, 0, 1, n_q, qp, L - 40)
    want = orc.gqa_attention(qp, k, v, v_lr, b[1], s, L - 40, n_q, n_kv)
    print("prefill", ctx.last_kernel(), orc.max_rel_error(got, want))
    pool.close()
if F32_ONLY:
    ctx.close()
    sys.exit(0)
# fused K / V projection + RoPE + append (tcgen05) and the tensor-core X * A projection
from paper_2602_01053_b200 import Adapters, Pool, Projection
for (L, d_model, n_kv, P) in [(200, 192, 1, 32), (300, 256, 2, 64)]:
    x = orc.round_bf16(orc.gaussian(L, d_model, 11, 1.0, np.float32))
    wk = orc.round_bf16(orc.gaussian(d_model, n_kv * 128, 12, 1.0 / np.sqrt(d_model), np.float32))
    wv = orc.round_bf16(orc.gaussian(d_model, n_kv * 128, 13, 1.0 / np.sqrt(d_model), np.float32))
    pool = Pool(ctx, "BaseLRShared", 1, n_kv, 128, d_model, 16, 1, max_tokens=L, dtype=abi.BF16, page_tokens=P)
    pj = Projection(ctx, 1, d_model, n_kv, 128, dtype=abi.BF16); pj.set_kv(0, wk, wv)
    ad = Adapters(ctx, 1, 1, d_model, 16, n_kv, 128, dtype=abi.BF16)
    A = orc.gaussian(d_model, 16, 14, 1.0 / np.sqrt(d_model), np.float32); ad.set_a(0, A)
    pool.append_tokens(L)
    pool.append_kv_project(pj, 0, 0, 0, x[:77]); pool.append_kv_project(pj, 0, 0, 77, x[77:])
    pool.append_lr_project(ad, 0, 0, 0, x)
    k = orc.apply_rope(orc.matmul(x, wk), n_kv, 128, 0)
    print("kv_project", ctx.last_kernel(), orc.max_rel_error(pool.key_view(0, 0), k), orc.max_rel_error(pool.value_view(0, 0), orc.matmul(x, wv)),
          "lr", orc.max_rel_error(pool.lr_view(0, 0), orc.matmul(x, A)))
    pool.close(); pj.close(); ad.close()
# large-score prefill: exercises the lazy-rescale / correction path of the tcgen05 kernel
from tests.cases import synthetic_layer
n_q, n_kv, d, r, L, L_c = 8, 2, 128, 16, 600, 200
q1, k, v, v_lr, b, s = synthetic_layer(orc, 21, L, 1, n_q, n_kv, d, r, 2, amp=25.0)
rnd = orc.round_bf16
k, v, v_lr = rnd(k), rnd(v), rnd(v_lr); b = [rnd(x) for x in b]
q = rnd(orc.gaussian(L_c, n_q * d, 4321, 25.0 / np.sqrt(d), np.float32))
pool = Pool(ctx, "BaseLRShared", 1, n_kv, d, 64, r, 2, max_tokens=L, dtype=abi.BF16)
ad = Adapters(ctx, 1, 2, 64, r, n_kv, d, dtype=abi.BF16)
pool.append_tokens(L)
pool.append_key(0, 0, 0, k); pool.append_value(0, 0, 0, v); pool.append_lr(0, 0, 0, v_lr)
for a_ in range(2):
    ad.set_b(0, a_, b[a_], 16.0)
got = pool.prefill(ad, 0, 0, n_q, q, L - L_c)
print("prefill amp 25", ctx.last_kernel(), orc.max_rel_error(got, orc.gqa_attention(q, k, v, v_lr, b[0], s, L - L_c, n_q, n_kv)))
pool.close(); ad.close()
a = np.random.default_rng(0).standard_normal((128, 128)).astype(np.float32)
bm = np.random.default_rng(1).standard_normal((128, 64)).astype(np.float32)
print("selftest", np.abs(ctx.selftest_umma(a, bm, True, a_in_tmem=True)).max() > 0)
ctx.close()
