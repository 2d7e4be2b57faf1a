"""fp32 mode (north star: <= 1e-4 on max_rel_error) at BASELINE size, through size-independent properties and sampled direct
comparisons with the reference path: one layer of cfg 2 over fp32 pages on fla_decode_f32 (16-key tiles, split-TF32 scores, P V on
bf16 planes), and a cfg-3-shaped prefill block on fla_prefill_split (bf16 planes of the fp32 rows on tcgen05, key splits of 4 096
keys merged by the decode epilogue).  bench.py's f32_mode leg compares whole layers / 259 rows in every run; this keeps the same
shapes inside `pytest -m gpu`.  Needs a B200."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

N_Q, N_KV, D, R, A, L, D_MODEL = 32, 8, 128, 16, 3, 32768, 256
TOL = 1e-4


@pytest.fixture(scope="module")
def ctx():
    from paper_2602_01053_b200 import Context
    c = Context(0)
    yield c
    c.close()


@pytest.fixture(scope="module")
def layer(orc):
    g = lambda rows, cols, key, scale: orc.gaussian(rows, cols, orc.child(2603, key), scale, np.float32)
    return dict(k=g(L, N_KV * D, 2, 1.0 / np.sqrt(D)), v=g(L, N_KV * D, 3, 1.0), lr=g(L, R, 4, 1.0),
                b=[g(R, N_KV * D, 20 + a, 0.02 / np.sqrt(R)) for a in range(A)],
                q=np.stack([g(1, N_Q * D, 30 + a, 1.0 / np.sqrt(D))[0] for a in range(A)]))


@pytest.fixture(scope="module")
def store(ctx, layer):
    from paper_2602_01053_b200 import Adapters, Pool, abi
    pool = Pool(ctx, "BaseLRShared", 1, N_KV, D, D_MODEL, R, A, max_tokens=L, dtype=abi.F32)
    ad = Adapters(ctx, 1, A, D_MODEL, R, N_KV, D, dtype=abi.F32)
    pool.append_tokens(L)
    pool.append_key(0, 0, 0, layer["k"]); pool.append_value(0, 0, 0, layer["v"]); pool.append_lr(0, 0, 0, layer["lr"])
    for a in range(A):
        ad.set_b(0, a, layer["b"][a], 16.0)
    yield pool, ad
    pool.close(); ad.close()


def head_slice(layer, orc, q_rows, kvh, a, offset):
    g = N_Q // N_KV
    cols = slice(kvh * D, (kvh + 1) * D)
    qh = np.ascontiguousarray(q_rows[:, kvh * g * D:(kvh + 1) * g * D])
    Lv = offset + q_rows.shape[0]
    return orc.gqa_attention(qh, np.ascontiguousarray(layer["k"][:Lv, cols]), np.ascontiguousarray(layer["v"][:Lv, cols]),
                             np.ascontiguousarray(layer["lr"][:Lv]), np.ascontiguousarray(layer["b"][a][:, cols]), 16.0 / R, offset, g, 1)


def test_full_size_fp32_decode(ctx, orc, layer, store):
    pool, ad = store
    g = N_Q // N_KV
    out = pool.decode(ad, 0, 1, list(range(A)), N_Q, layer["q"][None])[0]
    assert ctx.last_kernel() == "fla_decode_f32"
    for a, kvh in ((0, 0), (1, 3), (2, 7)):
        want = head_slice(layer, orc, layer["q"][a][None, :], kvh, a, L - 1)
        assert orc.max_rel_error(out[a][None, kvh * g * D:(kvh + 1) * g * D], want) <= TOL, (a, kvh)
    # the CUDA-core kernel (fp32 FFMA, policy 1) and the tensor-core kernel agree far inside the tolerance
    ctx.set_kernel_policy(1)
    try:
        ref = pool.decode(ad, 0, 1, list(range(A)), N_Q, layer["q"][None])[0]
        assert ctx.last_kernel() == "fla_paged_simt"
    finally:
        ctx.set_kernel_policy(0)
    assert orc.max_rel_error(out, ref) <= 2e-5
    # kv-head shards give the shard's slice (no communication inside attention)
    from paper_2602_01053_b200 import Adapters, Pool, abi
    kb, kn = 5, 2
    sp = Pool(ctx, "BaseLRShared", 1, N_KV, D, D_MODEL, R, A, max_tokens=L, dtype=abi.F32, kv_head_begin=kb, n_kv_local=kn)
    sa = Adapters(ctx, 1, A, D_MODEL, R, N_KV, D, kv_head_begin=kb, n_kv_local=kn, dtype=abi.F32)
    sp.append_tokens(L)
    sp.append_key(0, 0, 0, layer["k"]); sp.append_value(0, 0, 0, layer["v"]); sp.append_lr(0, 0, 0, layer["lr"])
    for a in range(A):
        sa.set_b(0, a, layer["b"][a], 16.0)
    q_local = np.ascontiguousarray(layer["q"][:, kb * g * D:(kb + kn) * g * D])
    got = sp.decode(sa, 0, 1, list(range(A)), N_Q, q_local[None])[0]
    assert orc.max_rel_error(got, out[:, kb * g * D:(kb + kn) * g * D]) <= 2e-5
    sp.close(); sa.close()


def test_full_size_fp32_prefill_on_tcgen05(ctx, orc, layer, store):
    """4 096 query rows at the end of the 32 768-token trajectory: eight key splits per row block, the last ones partly masked;
    sampled rows against the reference path (L_c = 1 per row), the whole block against the mma.sync TF32 kernel."""
    pool, ad = store
    L_c, off, agent = 4096, L - 4096, 1
    g = N_Q // N_KV
    q = orc.gaussian(L_c, N_Q * D, orc.child(2603, 77), 1.0 / np.sqrt(D), np.float32)
    out = pool.prefill(ad, 0, agent, N_Q, q, off)
    assert ctx.last_kernel() == "fla_prefill_split"
    rows = sorted({0, 1, L_c - 1} | set(np.random.default_rng(99).choice(L_c, size=12, replace=False).tolist()))
    for i, r in enumerate(rows):
        kvh = (3 * i) % N_KV
        want = head_slice(layer, orc, q[r:r + 1], kvh, agent, off + r)
        assert orc.max_rel_error(out[r:r + 1, kvh * g * D:(kvh + 1) * g * D], want) <= TOL, (r, kvh)
    ctx.set_kernel_policy(2)
    try:
        ref = pool.prefill(ad, 0, agent, N_Q, q, off)
        assert ctx.last_kernel() == "fla_prefill_f32"
    finally:
        ctx.set_kernel_policy(0)
    assert orc.max_rel_error(out, ref) <= 5e-5
    # a cold block (no prefix): rows attend only to themselves, most key splits of a row block are empty
    cold = pool.prefill(ad, 0, agent, N_Q, q[:512], 0)
    assert ctx.last_kernel() == "fla_prefill_split"
    for r, kvh in ((0, 2), (300, 6), (511, 1)):
        want = head_slice(layer, orc, q[r:r + 1], kvh, agent, r)
        assert orc.max_rel_error(cold[r:r + 1, kvh * g * D:(kvh + 1) * g * D], want) <= TOL, (r, kvh)
