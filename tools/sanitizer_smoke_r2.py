"""compute-sanitizer workload for the kernels added in round 2: the fused layer-step projections (step_partial / step_finish),
the dependent-launch chain with the prefetch before the wait, the one-round-trip merge, the key-side low-rank term
(qk projection, L_k tiles in fla_decode_tma and in the CUDA-core kernel), fp64 pages / the hidden cache / overwrite.
Run as  compute-sanitizer --tool memcheck|racecheck|synccheck python tools/sanitizer_smoke_r2.py"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from oracle import checker  # noqa: E402
import paper_2602_01053_b200 as pkg  # noqa: E402
from paper_2602_01053_b200 import Adapters, Pool, Projection, abi  # noqa: E402

orc = checker.oracle()
ctx = pkg.Context(0)
rnd = orc.round_bf16
g = lambda rows, cols, key, scale: rnd(orc.gaussian(rows, cols, orc.child(77, key), scale, np.float32))

# ---- fused layer-step chain: projections (2 launches) -> attention (prefetch before the wait) -> merge, 6 tokens x 2 layers
d_model, n_q, n_kv, d, r, A, P, L0, n_gen, n_layers = 256, 8, 2, 128, 16, 2, 32, 60, 6, 2
pool = Pool(ctx, "BaseLRShared", n_layers, n_kv, d, d_model, r, A, max_tokens=128, dtype=abi.BF16, page_tokens=P)
proj = Projection(ctx, n_layers, d_model, n_kv, d, dtype=abi.BF16)
ad = Adapters(ctx, n_layers, A, d_model, r, n_kv, d, dtype=abi.BF16)
x = g(L0 + n_gen, d_model, 1, 1.0)
ws = []
for l in range(n_layers):
    wq, wk, wv = g(d_model, n_q * d, 10 * l + 2, d_model ** -0.5), g(d_model, n_kv * d, 10 * l + 3, d_model ** -0.5), g(d_model, n_kv * d, 10 * l + 4, d_model ** -0.5)
    a_q, a_v = g(d_model, r, 10 * l + 5, d_model ** -0.5), g(d_model, r, 10 * l + 6, d_model ** -0.5)
    proj.set_kv(l, wk, wv); proj.set_q(l, n_q, wq); ad.set_a(l, a_v)
    bq = [g(r, n_q * d, 10 * l + 7 + a, 0.02) for a in range(A)]; bv = [g(r, n_kv * d, 10 * l + 9 + a, 0.02) for a in range(A)]
    for a in range(A):
        proj.set_q_lora(l, a, A, a_q, bq[a], 16.0); ad.set_b(l, a, bv[a], 16.0)
    ws.append((wq, wk, wv, a_q, a_v, bq, bv))
pool.append_tokens(L0)
for l in range(n_layers):
    pool.append_kv_project(proj, l, 0, 0, x[:L0]); pool.append_lr_project(ad, l, 0, 0, x[:L0])
xd = torch.from_numpy(x).cuda(); od = torch.zeros((n_layers, n_q * d), device="cuda")
for t in range(n_gen):
    pool.append_tokens(1)
    for l in range(n_layers):
        pool.step_layer_device(proj, ad, l, t % A, L0 + t, xd[L0 + t].data_ptr(), 1, d_model, n_q, od[l].data_ptr())
ctx.synchronize()
wq, wk, wv, a_q, a_v, bq, bv = ws[1]
row, agent = L0 + n_gen - 1, (n_gen - 1) % A
xs = x[:row + 1]
q = orc.apply_rope(orc.matmul(x[row:row + 1], wq) + np.float32(1.0) * orc.matmul(orc.matmul(x[row:row + 1], a_q), bq[agent]), n_q, d, row)
want = orc.gqa_attention(q, orc.apply_rope(orc.matmul(xs, wk), n_kv, d, 0), orc.matmul(xs, wv), orc.matmul(xs, a_v), bv[agent], 1.0, row, n_q, n_kv)
print("step_layer chain", ctx.last_kernel(), orc.max_rel_error(od[1].cpu().numpy()[None, :], want))
# per-layer decode launches back to back (prefetch before the wait, one-round-trip merge)
qd = torch.randn((n_layers, A, n_q * d), device="cuda") * (d ** -0.5); outd = torch.zeros_like(qd)
for _ in range(3):
    for l in range(n_layers):
        pool.decode_device(ad, l, l + 1, [0, 1], n_q, qd[l].data_ptr(), outd[l].data_ptr())
ctx.synchronize()
print("per-layer decode", ctx.last_kernel(), bool(torch.isfinite(outd).all()))
pool.close(); proj.close(); ad.close()

# ---- key-side low-rank term: tensor-core decode (rank_k 16) and the CUDA-core kernel (fp32 pages)
for dt, name in ((abi.BF16, "bf16"), (abi.F32, "f32")):
    L, r_k = 150, 16
    pool = Pool(ctx, "BaseLRShared", 1, n_kv, d, d_model, r, A, max_tokens=L, dtype=dt, page_tokens=32, rank_k=r_k)
    ad = Adapters(ctx, 1, A, d_model, r, n_kv, d, dtype=dt); ad.enable_key(r_k)
    k, v, v_lr, l_k = g(L, n_kv * d, 50, d ** -0.5), g(L, n_kv * d, 51, 1.0), g(L, r, 52, 1.0), g(L, r_k, 53, 1.0)
    pool.append_tokens(L); pool.append_key(0, 0, 0, k); pool.append_value(0, 0, 0, v); pool.append_lr(0, 0, 0, v_lr); pool.append_lk(0, 0, l_k)
    bv = [g(r, n_kv * d, 54 + a, 0.02) for a in range(A)]; bk = [g(r_k, n_kv * d, 56 + a, 0.1) for a in range(A)]
    for a in range(A):
        ad.set_b(0, a, bv[a], 16.0); ad.set_b_k(0, a, bk[a], 16.0)
    qh = g(A, n_q * d, 58, d ** -0.5)
    out = pool.decode(ad, 0, 1, list(range(A)), n_q, qh[None])
    keys = k + np.float32(1.0) * orc.matmul(l_k, bk[1])
    want = orc.gqa_attention(qh[1:2], keys, v, v_lr, bv[1], 1.0, L - 1, n_q, n_kv)
    print("key low-rank", name, ctx.last_kernel(), orc.max_rel_error(out[0, 1][None, :], want))
    pool.close(); ad.close()

# ---- hidden cache and fp64 pages (storage kernels of the SelectiveRecompute / KvStore<double> stores)
pool = Pool(ctx, "SelectiveRecompute", 2, 2, 8, 16, 0, 2, max_tokens=64, dtype=abi.F32, page_tokens=16)
rows = orc.gaussian(20, 16, 90, 1.0, np.float32)
pool.append_tokens(20)
assert pool._append(3, 0, 0, 0, rows) == 20
print("hidden cache rows", pool.rows(3, 0, 0))
pool.close()
ctx.close()
