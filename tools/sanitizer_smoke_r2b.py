"""compute-sanitizer workload for the kernels added late in round 2: the fp32-mode tcgen05 prefill (split_planes + fla_prefill_split
with several key splits, an empty split and a ragged last row block), the plane projections (pack_x_planes / pack_w_planes + the
GEMM kernel in query mode, K / V scatter), and the key-side low-rank term on fla_prefill_umma / fla_decode_umma.
Run as  LORAKV_SPLIT_KEYS=128 compute-sanitizer --tool memcheck|racecheck|synccheck python tools/sanitizer_smoke_r2b.py"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import checker  # noqa: E402
import paper_2602_01053_b200 as pkg  # noqa: E402
from paper_2602_01053_b200 import Adapters, Pool, Projection, abi  # noqa: E402

orc = checker.oracle()
ctx = pkg.Context(0)
g = lambda rows, cols, key, scale: orc.gaussian(rows, cols, orc.child(99, key), scale, np.float32)

# ---- fp32-mode prefill on tcgen05: 300 keys, 70 positions x group 4 = 280 rows (three row blocks, the last one ragged)
n_q, n_kv, d, r, A, L, L_c, d_model = 8, 2, 128, 16, 2, 300, 70, 256
for rank in (16, 0):
    pool = Pool(ctx, "BaseLRShared" if rank else "FullShared", 1, n_kv, d, d_model, rank, A, max_tokens=L, dtype=abi.F32, page_tokens=32)
    ad = Adapters(ctx, 1, A, d_model, max(rank, 1), n_kv, d, dtype=abi.F32)
    k, v, v_lr = g(L, n_kv * d, 1, d ** -0.5), g(L, n_kv * d, 2, 1.0), g(L, rank, 3, 1.0)
    b = [g(max(rank, 1), n_kv * d, 4 + a, 0.02) for a in range(A)]
    pool.append_tokens(L); pool.append_key(0, 0, 0, k); pool.append_value(0, 0, 0, v)
    if rank:
        pool.append_lr(0, 0, 0, v_lr)
    for a in range(A):
        ad.set_b(0, a, b[a], 16.0)
    q = g(L_c, n_q * d, 6, d ** -0.5)
    for off in (L - L_c, 40):
        got = pool.prefill(ad, 0, 1, n_q, q, off)
        want = orc.gqa_attention(q, k[:off + L_c], v[:off + L_c], v_lr[:off + L_c], b[1][:rank], 16.0 / max(rank, 1), off, n_q, n_kv)
        print("fp32 prefill", rank, off, ctx.last_kernel(), orc.max_rel_error(got, want))
    pool.close(); ad.close()

# ---- plane projections: 300 rows, K / V with rotation into fp32 pages, q with the adapter
x, wk, wv = g(L, d_model, 10, 1.0), g(d_model, n_kv * d, 11, d_model ** -0.5), g(d_model, n_kv * d, 12, d_model ** -0.5)
wq, a_q, b_q = g(d_model, n_q * d, 13, d_model ** -0.5), g(d_model, 8, 14, d_model ** -0.5), g(8, n_q * d, 15, 0.1)
pool = Pool(ctx, "FullShared", 1, n_kv, d, d_model, 0, 1, max_tokens=L, dtype=abi.F32, page_tokens=64)
proj = Projection(ctx, 1, d_model, n_kv, d, dtype=abi.F32)
proj.set_kv(0, wk, wv); proj.set_q(0, n_q, wq); proj.set_q_lora(0, 0, 1, a_q, b_q, 16.0)
pool.append_tokens(L)
assert pool.append_kv_project(proj, 0, 0, 0, x) == L
print("plane projections", ctx.last_kernel(), orc.max_rel_error(pool.key_view(0, 0), orc.apply_rope(orc.matmul(x, wk), n_kv, d, 0)),
      orc.max_rel_error(pool.value_view(0, 0), orc.matmul(x, wv)))
got = proj.query(0, 0, 5, x, n_q * d, rope=True)
want = orc.apply_rope(orc.matmul(x, wq) + np.float32(2.0) * orc.matmul(orc.matmul(x, a_q), b_q), n_q, d, 5)
print("plane query", ctx.last_kernel(), orc.max_rel_error(got, want))
pool.close(); proj.close()

# ---- key-side low-rank term on the tcgen05 kernels (bf16 pages): 40 decode rows per kv head, a 150-row prefill block
rnd = orc.round_bf16
A, L, r_k = 10, 260, 32
pool = Pool(ctx, "BaseLRShared", 1, n_kv, d, d_model, r, A, max_tokens=L, dtype=abi.BF16, page_tokens=32, rank_k=r_k)
ad = Adapters(ctx, 1, A, d_model, r, n_kv, d, dtype=abi.BF16); ad.enable_key(r_k)
k, v, v_lr, l_k = rnd(g(L, n_kv * d, 20, d ** -0.5)), rnd(g(L, n_kv * d, 21, 1.0)), rnd(g(L, r, 22, 1.0)), rnd(g(L, r_k, 23, 1.0))
pool.append_tokens(L); pool.append_key(0, 0, 0, k); pool.append_value(0, 0, 0, v); pool.append_lr(0, 0, 0, v_lr); pool.append_lk(0, 0, l_k)
bv = [rnd(g(r, n_kv * d, 30 + a, 0.02)) for a in range(A)]; bk = [rnd(g(r_k, n_kv * d, 50 + a, 0.1)) for a in range(A)]
for a in range(A):
    ad.set_b(0, a, bv[a], 16.0); ad.set_b_k(0, a, bk[a], 32.0)
qh = rnd(g(A, n_q * d, 70, d ** -0.5))
out = pool.decode(ad, 0, 1, list(range(A)), n_q, qh[None])
keys = k + np.float32(1.0) * orc.matmul(l_k, bk[3])
print("key low-rank decode", ctx.last_kernel(), orc.max_rel_error(out[0, 3][None, :], orc.gqa_attention(qh[3:4], keys, v, v_lr, bv[3], 1.0, L - 1, n_q, n_kv)))
qb = rnd(g(150, n_q * d, 71, d ** -0.5))
got = pool.prefill(ad, 0, 3, n_q, qb, L - 150)
print("key low-rank prefill", ctx.last_kernel(), orc.max_rel_error(got, orc.gqa_attention(qb, keys, v, v_lr, bv[3], 1.0, L - 150, n_q, n_kv)))
pool.close(); ad.close()

# ---- BaseShared batch in one launch: per-entry V_lr tiles, 32-key tiles on the multi-warp workers (40 rows per kv head)
A, L = 10, 200
pool = Pool(ctx, "BaseShared", 1, n_kv, d, d_model, r, A, max_tokens=L, dtype=abi.BF16, page_tokens=32)
ad = Adapters(ctx, 1, A, d_model, r, n_kv, d, dtype=abi.BF16)
k, v = rnd(g(L, n_kv * d, 80, d ** -0.5)), rnd(g(L, n_kv * d, 81, 1.0))
lrs = [rnd(g(L, r, 82 + a, 1.0)) for a in range(A)]
bv = [rnd(g(r, n_kv * d, 100 + a, 0.02)) for a in range(A)]
pool.append_tokens(L); pool.append_key(0, 0, 0, k); pool.append_value(0, 0, 0, v)
for a in range(A):
    pool.append_lr(0, a, 0, lrs[a]); ad.set_b(0, a, bv[a], 16.0)
qh = rnd(g(A, n_q * d, 120, d ** -0.5))
out = pool.decode(ad, 0, 1, list(range(A)), n_q, qh[None])
print("BaseShared batch", ctx.last_kernel(), orc.max_rel_error(out[0, 7][None, :], orc.gqa_attention(qh[7:8], k, v, lrs[7], bv[7], 1.0, L - 1, n_q, n_kv)))
pool.close(); ad.close()
ctx.close()
