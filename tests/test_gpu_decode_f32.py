"""fp32 mode of the decode path (fla_decode_f32: TMA bulk-copy rings over swizzled fp32 pages + 3 x TF32 mma.sync)
against the CPU oracle through the C ABI.  Oracle = gqa_attention per (agent, layer) (attention.hpp:332-363), as
engine.hpp:440-443 calls it; tolerance 1e-4 on max_rel_error (BASELINE.json north_star, fp32 mode; cli.cpp:94).
Needs a B200."""
import numpy as np
import pytest

from tests.test_gpu_pool import build_pool

pytestmark = pytest.mark.gpu

TOL = 1e-4


@pytest.fixture(scope="module")
def ctx():
    from paper_2602_01053_b200 import Context
    c = Context(0)
    yield c
    c.close()


def check(ctx, orc, pool, ad, layers, batch, n_q, n_kv, L, amp_note=""):
    n_layers = len(layers)
    qs = np.stack([np.stack([layers[l][0][a][0] for a in batch]) for l in range(n_layers)])
    outs = {}
    for policy, kernel in ((0, "fla_decode_f32"), (1, "fla_paged_simt")):
        ctx.set_kernel_policy(policy)
        out = pool.decode(ad, 0, n_layers, batch, n_q, qs)
        assert ctx.last_kernel() == kernel, (policy, ctx.last_kernel())
        outs[policy] = out
        worst = 0.0
        for l in range(n_layers):
            q, k, v, v_lr, b, s = layers[l]
            for i, a in enumerate(batch):
                bb = b[a] if len(b) else np.zeros((0, k.shape[1]), np.float32)
                want = orc.gqa_attention(q[a], k, v, v_lr, bb, s, L - 1, n_q, n_kv)
                worst = max(worst, orc.max_rel_error(out[l, i][None, :], want))
        assert worst <= TOL, (policy, worst, amp_note)
    ctx.set_kernel_policy(0)
    assert orc.max_rel_error(outs[0].reshape(1, -1), outs[1].reshape(1, -1)) <= TOL


# n_q, n_kv, d, r, agents, L, P, layers
SHAPES = [
    (8, 2, 128, 16, 3, 1000, 64, 2),    # 12 rows: one warp per worker (the Llama cfg-2 row count)
    (32, 8, 128, 16, 3, 257, 64, 1),    # Llama head counts
    (8, 2, 128, 64, 8, 777, 32, 1),     # 32 rows, rank 64: two warps per worker
    (4, 1, 128, 32, 16, 530, 64, 1),    # 64 rows, rank 32: four warps per worker
    (16, 2, 64, 8, 12, 300, 16, 1),     # 96 rows, d = 64, rank 8 padded to 16
    (8, 1, 128, 4, 20, 211, 8, 1),      # 160 rows: two 128-row blocks; 8-token pages
    (4, 2, 64, 24, 2, 130, 128, 3),     # rank 24 padded to 32, 128-token pages, 3 layers
    (4, 2, 128, 0, 2, 333, 64, 1),      # rank 0: plain attention (FullShared contents)
]


@pytest.mark.parametrize("n_q,n_kv,d,r,A,L,P,n_layers", SHAPES)
def test_decode_f32_matches_reference_path(ctx, orc, n_q, n_kv, d, r, A, L, P, n_layers):
    from paper_2602_01053_b200 import abi
    scheme = "BaseLRShared" if r > 0 else "FullShared"
    pool, ad, layers = build_pool(ctx, orc, scheme, abi.F32, 2000 + L, L, n_layers, n_q, n_kv, d, r, A, P=P)
    check(ctx, orc, pool, ad, layers, list(range(A)), n_q, n_kv, L)
    pool.close()


@pytest.mark.parametrize("L", [1, 7, 8, 9, 63, 64, 65, 4099])
def test_decode_f32_ragged_lengths(ctx, orc, L):
    """Single-token caches, tiles and pages that end mid-way; keys >= L must contribute exactly 0."""
    from paper_2602_01053_b200 import abi
    n_q, n_kv, d, r, A = 8, 2, 128, 16, 3
    pool, ad, layers = build_pool(ctx, orc, "BaseLRShared", abi.F32, 70 + L, L, 1, n_q, n_kv, d, r, A, P=32)
    check(ctx, orc, pool, ad, layers, [2, 0, 1, 1], n_q, n_kv, L)
    pool.close()


@pytest.mark.parametrize("amp", [5.0, 25.0])
def test_decode_f32_large_scores(ctx, orc, amp):
    """fuzz.hpp:30,40-43 amplitudes: scores of several hundred, near exp underflow -- the split-TF32 products must
    keep the score error far below one ulp of the softmax."""
    from paper_2602_01053_b200 import Adapters, Pool, abi
    from tests.cases import synthetic_layer
    n_q, n_kv, d, r, A, L = 8, 2, 128, 16, 3, 600
    pool = Pool(ctx, "BaseLRShared", 1, n_kv, d, 64, r, A, max_tokens=L, dtype=abi.F32)
    ad = Adapters(ctx, 1, A, 64, r, n_kv, d, dtype=abi.F32)
    q, k, v, v_lr, b, s = synthetic_layer(orc, 4242, L, 1, n_q, n_kv, d, r, A, amp=amp)
    pool.append_tokens(L)
    pool.append_key(0, 0, 0, k); pool.append_value(0, 0, 0, v); pool.append_lr(0, 0, 0, v_lr)
    for a in range(A):
        ad.set_b(0, a, b[a], 16.0)
    check(ctx, orc, pool, ad, [(q, k, v, v_lr, b, s)], list(range(A)), n_q, n_kv, L, amp_note=f"amp {amp}")
    pool.close()


# ---- prefill blocks in fp32 mode (fla_prefill_f32: the same split-TF32 fragments as a flash-attention forward) ----------
def run_prefill(ctx, orc, n_q, n_kv, d, r, L, L_c, offsets, P, seed, scheme="BaseLRShared", amp=1.0, agent=1, split_keys=0):
    from paper_2602_01053_b200 import abi
    A = 2
    pool, ad, layers = build_pool(ctx, orc, scheme, abi.F32, seed, L, 1, n_q, n_kv, d, r, A, P=P)
    _, k, v, v_lr, b, s = layers[0]
    q = orc.gaussian(L_c, n_q * d, seed + 77, amp / np.sqrt(d), np.float32)
    bb = b[agent] if r > 0 else np.zeros((0, n_kv * d), np.float32)
    # blocks of >= 128 query rows per kv head run on the tensor-core plane kernel (fla_prefill_split), smaller ones (and
    # policy 2) on the mma.sync TF32 kernel
    fast = "fla_prefill_split" if L_c * (n_q // n_kv) >= 128 else "fla_prefill_f32"
    ctx.set_prefill_split_keys(split_keys)
    for off in offsets:
        want = orc.gqa_attention(q, k, v, v_lr, bb, s, off, n_q, n_kv)
        for policy, kernel in ((2, "fla_prefill_f32"), (0, fast)):
            ctx.set_kernel_policy(policy)
            got = pool.prefill(ad, 0, agent, n_q, q, off)
            assert ctx.last_kernel() == kernel, (policy, ctx.last_kernel())
            err = orc.max_rel_error(got, want)
            assert err <= TOL, (off, kernel, err)
        ctx.set_kernel_policy(1)
        ref = pool.prefill(ad, 0, agent, n_q, q, off)
        assert ctx.last_kernel() == "fla_paged_simt"
        ctx.set_kernel_policy(0)
        assert orc.max_rel_error(got, ref) <= TOL
    ctx.set_prefill_split_keys(0)
    pool.close()


PREFILL_SHAPES = [
    (8, 2, 128, 16, 300, 40, (260, 0, 131), 64),       # group 4 -> 32 positions per CTA (the Llama mapping)
    (4, 2, 64, 8, 333, 77, (256, 100, 0), 64),          # d = 64, rank 8 padded to 16, group 2
    (4, 4, 128, 32, 700, 300, (400, 0), 32),            # group 1: 128 positions per CTA, several row blocks
    (16, 2, 128, 64, 520, 130, (390, 17), 128),         # group 8, rank 64, 128-token pages
    (8, 2, 128, 0, 450, 64, (386, 0), 16),              # rank 0 (FullShared), 16-token pages
    (32, 8, 128, 16, 1100, 96, (1004, 500), 64),        # Llama head counts
    (8, 2, 128, 16, 129, 2, (127, 0), 8),               # two query rows, 8-token pages
    (6, 2, 64, 16, 200, 50, (150, 3), 64),              # group 3: a position's heads straddle 16-row warps
]


@pytest.mark.parametrize("n_q,n_kv,d,r,L,L_c,offsets,P", PREFILL_SHAPES)
def test_prefill_f32_matches_reference_path(ctx, orc, n_q, n_kv, d, r, L, L_c, offsets, P):
    run_prefill(ctx, orc, n_q, n_kv, d, r, L, L_c, offsets, P, seed=800 + L, scheme="FullShared" if r == 0 else "BaseLRShared")


@pytest.mark.parametrize("split_keys", [64, 128, 192])
@pytest.mark.parametrize("n_q,n_kv,d,r,L,L_c,offsets,P", PREFILL_SHAPES[:6] + [PREFILL_SHAPES[7]])
def test_prefill_f32_key_splits(ctx, orc, n_q, n_kv, d, r, L, L_c, offsets, P, split_keys):
    """The tensor-core plane kernel with many key splits per row block (one to three 64-key tiles per split): splits that end
    inside a row's causal range, splits wholly beyond it (empty partials), rows whose first visible key lies in a later tile of
    their split, ragged last row blocks -- all combined by the merge epilogue."""
    run_prefill(ctx, orc, n_q, n_kv, d, r, L, L_c, offsets, P, seed=900 + L, scheme="FullShared" if r == 0 else "BaseLRShared",
                split_keys=split_keys)


@pytest.mark.parametrize("amp", [5.0, 25.0])
def test_prefill_f32_large_scores(ctx, orc, amp):
    run_prefill(ctx, orc, 8, 2, 128, 16, 600, 200, (400,), 64, seed=4321, amp=amp, agent=0)
    run_prefill(ctx, orc, 8, 2, 128, 16, 600, 200, (400, 0), 64, seed=4321, amp=amp, agent=0, split_keys=128)


def test_prefill_f32_masked_keys_contribute_exactly_zero(ctx, orc):
    """test_attention.cpp:144-175 through the fp32 prefill: keys beyond every row's causal boundary hold 1e6-sized
    values and must not change a single bit of the output."""
    from paper_2602_01053_b200 import Adapters, Pool, abi
    from tests.cases import synthetic_layer
    n_q, n_kv, d, r, L, L_c, off = 8, 2, 128, 16, 400, 50, 100       # rows see keys <= 149; 150..399 are hidden
    _, k, v, v_lr, b, s = synthetic_layer(orc, 33, L, 1, n_q, n_kv, d, r, 2)
    q = orc.gaussian(L_c, n_q * d, 99, 1.0 / np.sqrt(d), np.float32)
    outs = []
    for poison in (False, True):
        kk, vv, ll = k.copy(), v.copy(), v_lr.copy()
        if poison:
            kk[off + L_c:] = 1e6; vv[off + L_c:] = -1e6; ll[off + L_c:] = 1e6
        pool = Pool(ctx, "BaseLRShared", 1, n_kv, d, 64, r, 2, max_tokens=L, dtype=abi.F32)
        ad = Adapters(ctx, 1, 2, 64, r, n_kv, d, dtype=abi.F32)
        pool.append_tokens(L)
        pool.append_key(0, 0, 0, kk); pool.append_value(0, 0, 0, vv); pool.append_lr(0, 0, 0, ll)
        for a in range(2):
            ad.set_b(0, a, b[a], 16.0)
        for policy, kernel in ((0, "fla_prefill_split"), (2, "fla_prefill_f32")):
            ctx.set_kernel_policy(policy)
            outs.append(pool.prefill(ad, 0, 1, n_q, q, off))
            assert ctx.last_kernel() == kernel
        ctx.set_kernel_policy(0)
        pool.close(); ad.close()
    assert np.array_equal(outs[0], outs[2]) and np.array_equal(outs[1], outs[3])


@pytest.mark.parametrize("L_c,kernel", [(16, "fla_prefill_f32"), (64, "fla_prefill_split")])
def test_prefill_f32_long_rows_stay_at_fp32_accuracy(ctx, orc, L_c, kernel):
    """A 32K-token row is 4096 key tiles.  Tensor-core MMAs add into their accumulator with truncation, a bias that grows
    linearly with the chain (2e-4 at this length when the running sums lived in the MMA accumulators); the kernels keep the
    running sums in ordinary fp32 adds instead.  Checked against the float64 reference path, far inside the 1e-4 contract."""
    from paper_2602_01053_b200 import Adapters, Pool, abi
    from tests.cases import synthetic_layer
    n_q, n_kv, d, r, A, L = 4, 2, 128, 16, 2, 32768
    _, k, v, v_lr, b, s = synthetic_layer(orc, 11, L, 1, n_q, n_kv, d, r, A)
    q = orc.gaussian(L_c, n_q * d, 99, 1.0 / np.sqrt(d), np.float32)
    pool = Pool(ctx, "BaseLRShared", 1, n_kv, d, 64, r, A, max_tokens=L, dtype=abi.F32)
    ad = Adapters(ctx, 1, A, 64, r, n_kv, d, dtype=abi.F32)
    pool.append_tokens(L)
    pool.append_key(0, 0, 0, k); pool.append_value(0, 0, 0, v); pool.append_lr(0, 0, 0, v_lr)
    for a in range(A):
        ad.set_b(0, a, b[a], 16.0)
    got = pool.prefill(ad, 0, 1, n_q, q, L - L_c)
    assert ctx.last_kernel() == kernel
    f64 = lambda x: np.asarray(x, np.float64)
    want = orc.gqa_attention(f64(q), f64(k), f64(v), f64(v_lr), f64(b[1]), float(s), L - L_c, n_q, n_kv)
    err = float(np.max(np.abs(f64(got) - want)) / np.max(np.abs(want)))
    # the plane kernel bounds its truncating accumulate chains by key splits of 4096 (fla_prefill_split.cu)
    assert err <= (2e-5 if kernel == "fla_prefill_f32" else 4e-5), err
    pool.close(); ad.close()
