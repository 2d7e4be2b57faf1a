import sys, numpy as np
sys.path.insert(0, ".")
from oracle import checker
import paper_2602_01053_b200 as pkg
from paper_2602_01053_b200 import abi
from tests.test_gpu_pool import build_pool
orc = checker.oracle(); ctx = pkg.Context(0)
for (n_q, n_kv, d, r, A, L, P) in ((8, 2, 128, 16, 3, 500, 64), (8, 2, 128, 32, 8, 300, 32), (4, 1, 128, 16, 20, 211, 16)):
    pool, ad, layers = build_pool(ctx, orc, "BaseLRShared", abi.F32, 7, L, 2, n_q, n_kv, d, r, A, P=P)
    qs = np.stack([np.stack([layers[l][0][a][0] for a in range(A)]) for l in range(2)])
    out = pool.decode(ad, 0, 2, list(range(A)), n_q, qs)
    q, k, v, v_lr, b, s = layers[1]
    want = orc.gqa_attention(q[1], k, v, v_lr, b[1], s, L - 1, n_q, n_kv)
    print("f32 decode", ctx.last_kernel(), A * n_q // n_kv, "rows", orc.max_rel_error(out[1, 1][None, :], want))
    pool.close(); ad.close()
ctx.close()
