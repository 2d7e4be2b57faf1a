"""fp32-mode prefill on the plane kernel: accuracy of a long row against float64 and time per layer (tools, not a test).
usage: python tools/probe_prefill_split.py [L] [L_c]   (LORAKV_SPLIT_KEYS=... to vary the split)"""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_01053_b200 import Adapters, Context, Pool, abi
from oracle import checker
from tests.cases import synthetic_layer

L = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
L_c = int(sys.argv[2]) if len(sys.argv) > 2 else 64
orc = checker.oracle()
ctx = Context(0)
n_q, n_kv, d, r, A = 4, 2, 128, 16, 2
_, k, v, v_lr, b, s = synthetic_layer(orc, 11, L, 1, n_q, n_kv, d, r, A)
q = orc.gaussian(L_c, n_q * d, 99, 1.0 / np.sqrt(d), np.float32)
pool = Pool(ctx, "BaseLRShared", 1, n_kv, d, 64, r, A, max_tokens=L, dtype=abi.F32)
ad = Adapters(ctx, 1, A, 64, r, n_kv, d, dtype=abi.F32)
pool.append_tokens(L)
pool.append_key(0, 0, 0, k); pool.append_value(0, 0, 0, v); pool.append_lr(0, 0, 0, v_lr)
for a in range(A):
    ad.set_b(0, a, b[a], 16.0)
f64 = lambda x: np.asarray(x, np.float64)
want = orc.gqa_attention(f64(q), f64(k), f64(v), f64(v_lr), f64(b[1]), float(s), L - L_c, n_q, n_kv)
for policy in (0, 2):
    ctx.set_kernel_policy(policy)
    got = pool.prefill(ad, 0, 1, n_q, q, L - L_c)
    err = float(np.max(np.abs(f64(got) - want)) / np.max(np.abs(want)))
    bias = float(np.mean((f64(got) - want) * np.sign(want)) / np.mean(np.abs(want)))
    print(f"split_keys={os.environ.get('LORAKV_SPLIT_KEYS', 'default')} L={L} L_c={L_c} {ctx.last_kernel()}: max_rel_err {err:.3e}  signed shrink {bias:.3e}")
