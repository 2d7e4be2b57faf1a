import numpy as np, sys
sys.path.insert(0, "/root/repo")
from oracle import checker
import paper_2602_01053_b200 as pkg
from paper_2602_01053_b200 import abi
from tests.test_gpu_pool import build_pool
orc = checker.oracle()
ctx = pkg.Context(0)
# decode MW=1 and MW=2/KT=2, prefill umma, lr_project, selftest
for (n_q, n_kv, d, r, A, L, P) in [(8, 2, 128, 16, 3, 200, 64), (8, 2, 128, 32, 8, 150, 32), (16, 2, 64, 8, 12, 100, 16)]:
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
a = np.random.default_rng(0).standard_normal((128, 128)).astype(np.float32)
bm = np.random.default_rng(1).standard_normal((128, 64)).astype(np.float32)
print("selftest", np.abs(ctx.selftest_umma(a, bm, True, a_in_tmem=True)).max() > 0)
ctx.close()
