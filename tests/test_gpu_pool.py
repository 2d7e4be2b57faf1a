"""Paged cache pool + device-resident attention against the CPU oracle, through the C ABI.
Mirrors the reference's tests/test_kvcache.cpp (bookkeeping is bit-exact) and the engine's use of
gqa_attention (engine.hpp:440-443).  Needs a B200."""
import numpy as np
import pytest

from tests.cases import synthetic_layer

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    from paper_2602_01053_b200 import Context
    c = Context(0)
    yield c
    c.close()


def fill_rows(rows, cols, tag):
    return (tag + np.arange(rows * cols, dtype=np.float64)).reshape(rows, cols).astype(np.float32)


class PageModel:
    """CPU model of the page table (the reference has no pages): logical row ->
    (row // P, row % P) -- oracle orc_page_of -- and physical ids handed out in first-touch order
    within one page space shared by the sets (agents) of a scheme."""

    def __init__(self, orc, P):
        self.orc, self.P, self.next, self.tables = orc, P, 0, {}

    def touch(self, set_id, row_end):
        tab = self.tables.setdefault(set_id, [])
        if row_end <= 0:
            return
        last_page, _ = self.orc.page_of(row_end - 1, self.P)
        while len(tab) <= last_page:
            tab.append(self.next)
            self.next += 1


@pytest.mark.parametrize("scheme", ["NonShared", "FullShared", "BaseShared", "BaseLRShared"])
def test_store_bookkeeping_is_bit_exact(ctx, orc, scheme):
    """Random append traffic: rows, views, bytes, seen and page tables vs the oracle's KvStore."""
    from paper_2602_01053_b200 import Pool, abi
    n_layers, n_kv, d, r, N, P = 2, 2, 8, 4, 3, 16
    pool = Pool(ctx, scheme, n_layers, n_kv, d, 32, r, N, max_tokens=1024, dtype=abi.F32, page_tokens=P)
    st = orc.store(scheme, n_layers, n_kv * d, 32, r, N, np.float32)
    kv_model, lr_model = PageModel(orc, P), PageModel(orc, P)
    rng = np.random.default_rng(11)
    length = 0
    for step in range(14):
        n = int(rng.integers(1, 40)); agent = int(rng.integers(0, N))
        pool.append_tokens(n); st.append_tokens(n)
        assert pool.plan_step(agent, 0) == orc.plan_core(scheme, st.length(), st.seen(agent), 0)
        for layer in range(n_layers):
            have = st.key_view(layer, agent).shape[0]
            begin = max(0, have - int(rng.integers(0, 5)))
            rows = rng.standard_normal((length + n - begin, n_kv * d)).astype(np.float32)
            skip, add = orc.append_fww(have, begin, rows.shape[0])
            assert pool.append_key(layer, agent, begin, rows) == add
            assert pool.append_value(layer, agent, begin, rows + 1) == add
            st.append_key(layer, agent, begin, rows); st.append_value(layer, agent, begin, rows + 1)
            kv_model.touch(agent if scheme == "NonShared" else 0, have + add)
            if scheme in ("BaseShared", "BaseLRShared"):
                lhave = st.lr_view(layer, agent).shape[0]
                lbegin = max(0, lhave - int(rng.integers(0, 3)))
                lr = rng.standard_normal((length + n - lbegin, r)).astype(np.float32)
                pool.append_lr(layer, agent, lbegin, lr); st.append_lr(layer, agent, lbegin, lr)
                lr_model.touch(agent if scheme == "BaseShared" else 0, st.lr_view(layer, agent).shape[0])
        pool.mark_seen(agent); st.mark_seen(agent)
        length += n
        assert pool.length() == st.length()
        assert pool.bytes() == st.bytes()
        assert pool.allocated_elements() == st.allocated_elements()
        for a in range(N):
            assert pool.seen(a) == st.seen(a)
            for layer in range(n_layers):
                assert np.array_equal(pool.key_view(layer, a), st.key_view(layer, a))
                assert np.array_equal(pool.value_view(layer, a), st.value_view(layer, a))
                assert np.array_equal(pool.lr_view(layer, a), st.lr_view(layer, a))
            assert pool.page_table(abi.KEY, a).tolist() == kv_model.tables.get(a if scheme == "NonShared" else 0, [])
            if scheme in ("BaseShared", "BaseLRShared"):
                assert pool.page_table(abi.LR, a).tolist() == lr_model.tables.get(a if scheme == "BaseShared" else 0, [])
    pool.close()


def test_first_writer_wins_and_errors(ctx, orc, golden):
    """test_kvcache.cpp:116-152,266-277 on the device pool."""
    from paper_2602_01053_b200 import LorakvError, Pool, abi
    pool = Pool(ctx, "BaseShared", 1, 1, 4, 8, 2, 3, max_tokens=64, page_tokens=8)
    pool.append_tokens(6)
    base0 = fill_rows(6, 4, 0.0)
    pool.append_key(0, 0, 0, base0); pool.append_value(0, 0, 0, base0)
    pool.append_lr(0, 0, 0, fill_rows(6, 2, 10.0)); pool.mark_seen(0)
    base1 = fill_rows(6, 4, 500.0)
    assert pool.append_key(0, 1, 0, base1) == 0 and pool.append_value(0, 1, 0, base1) == 0
    pool.append_lr(0, 1, 0, fill_rows(6, 2, 20.0)); pool.mark_seen(1)
    assert pool.value_view(0, 1)[0, 0] == 0.0 and pool.key_view(0, 1)[5, 3] == base0[5, 3]
    assert pool.lr_view(0, 1)[0, 0] == 20.0 and pool.lr_view(0, 0)[0, 0] == 10.0
    with pytest.raises(LorakvError, match="gap") as e:
        pool.append_value(0, 0, 9, fill_rows(1, 4, 0.0))
    assert str(e.value) == "KvStore: value append leaves a gap at row 6"
    with pytest.raises(LorakvError):
        pool.seen(7)
    with pytest.raises(LorakvError, match="capacity"):
        pool.append_key(0, 0, 6, fill_rows(100, 4, 0.0))
    fs = Pool(ctx, "FullShared", 1, 1, 4, 8, 0, 2, max_tokens=16)
    with pytest.raises(LorakvError, match="no LR cache"):
        fs.append_lr(0, 0, 0, np.zeros((1, 0), np.float32))
    fs.append_tokens(4)
    fs.append_key(0, 0, 0, fill_rows(4, 4, 0.0)); fs.append_value(0, 0, 0, fill_rows(4, 4, 0.0))
    before = fs.bytes()
    fs.append_key(0, 1, 0, fill_rows(4, 4, 9.0)); fs.append_value(0, 1, 0, fill_rows(4, 4, 9.0))
    assert fs.bytes() == before and fs.value_view(0, 1)[0, 0] == 0.0
    assert fs.lr_view(0, 0).shape == (4, 0)


def test_byte_ratio_identities(ctx, golden):
    """test_kvcache.cpp:189-240 with the reference's byte counts from tests/golden (float64 there;
    the identities are ratios, so the fp32 pool is compared after scaling by sizeof)."""
    from paper_2602_01053_b200 import Pool
    L, N = 24, 3
    for row in golden["tables"]["store_bytes"]:
        r, d_out = row["r"], row["d_out"]
        got = {}
        for scheme in ("NonShared", "BaseShared", "BaseLRShared", "FullShared"):
            pool = Pool(ctx, scheme, 2, 1, d_out, 4 * d_out, r, N, max_tokens=L, page_tokens=8)
            pool.append_tokens(L)
            for layer in range(2):
                kv = fill_rows(L, d_out, 1000.0 * layer)
                for a in (range(N) if scheme == "NonShared" else (0,)):
                    pool.append_key(layer, a, 0, kv); pool.append_value(layer, a, 0, kv)
                lr = fill_rows(L, r, 77.0 + layer)
                if scheme == "BaseShared":
                    for a in range(N):
                        pool.append_lr(layer, a, 0, lr)
                if scheme == "BaseLRShared":
                    pool.append_lr(layer, 0, 0, lr)
            got[scheme] = pool.bytes()
            assert {k: 2 * v for k, v in got[scheme].items()} == row["bytes"][scheme]   # f32 vs f64
            assert pool.allocated_elements() == row["elements"][scheme]
            pool.close()
        ns, bs, blr, fs = got["NonShared"], got["BaseShared"], got["BaseLRShared"], got["FullShared"]
        assert (bs["value"] + bs["lr"]) * N * d_out == ns["value"] * (d_out + N * r)
        assert (blr["value"] + blr["lr"]) * N * d_out == ns["value"] * (d_out + r)
        assert fs["value"] * N == ns["value"] and blr["key"] * N == ns["key"]


def build_pool(ctx, orc, scheme, dtype, seed, L, n_layers, n_q, n_kv, d, r, n_agents, d_model=64, P=0,
               project=False):
    """Fill a pool layer by layer from SURVEY 8(d) synthetic inputs; returns everything the oracle needs."""
    from paper_2602_01053_b200 import Adapters, Pool, abi
    bf16 = dtype == abi.BF16
    rnd = (lambda a: orc.round_bf16(a)) if bf16 else (lambda a: a)
    pool = Pool(ctx, scheme, n_layers, n_kv, d, d_model, r, n_agents, max_tokens=L + 8, dtype=dtype, page_tokens=P)
    ad = Adapters(ctx, n_layers, n_agents, d_model, r, n_kv, d, dtype=dtype) if r > 0 else None
    pool.append_tokens(L)
    layers = []
    for layer in range(n_layers):
        q, k, v, v_lr, b, s = synthetic_layer(orc, seed + layer, L, 1, n_q, n_kv, d, r, n_agents)
        q = [rnd(x) for x in q]; k, v = rnd(k), rnd(v); b = [rnd(x) for x in b]
        pool.append_key(layer, 0, 0, k); pool.append_value(layer, 0, 0, v)
        if r > 0:
            if project:
                x = rnd(orc.gaussian(L, d_model, orc.child(seed + layer, 6), 1.0, np.float32))
                A = rnd(orc.gaussian(d_model, r, orc.child(seed + layer, 7), 1.0 / np.sqrt(d_model), np.float32))
                ad.set_a(layer, A)
                pool.append_lr_project(ad, layer, 0, 0, x)
                v_lr = orc.matmul(x, A)
            else:
                v_lr = rnd(v_lr)
                pool.append_lr(layer, 0, 0, v_lr)
            for a in range(n_agents):
                ad.set_b(layer, a, b[a], 16.0)
        layers.append((q, k, v, v_lr, b, s))
    return pool, ad, layers


@pytest.mark.parametrize("dtype_name,tol", [("F32", 1e-4), ("BF16", 2e-2)])
def test_tiny_config_decode_matches_reference_path(ctx, orc, dtype_name, tol):
    """BASELINE.json configs[0]: 4 q / 2 kv heads, d=64, r=8, 2 agents, L=512, decode.  Oracle =
    gqa_attention per (agent, layer) (attention.hpp:332), which is what engine.hpp:440-443 calls."""
    from paper_2602_01053_b200 import abi
    dtype = getattr(abi, dtype_name)
    L, n_layers, n_q, n_kv, d, r, A = 512, 2, 4, 2, 64, 8, 2
    pool, ad, layers = build_pool(ctx, orc, "BaseLRShared", dtype, 42, L, n_layers, n_q, n_kv, d, r, A)
    for policy in (1, 0):
        ctx.set_kernel_policy(policy)
        qs = np.stack([np.stack([layers[l][0][a][0] for a in range(A)]) for l in range(n_layers)])
        out = pool.decode(ad, 0, n_layers, [0, 1], n_q, qs)
        for l in range(n_layers):
            q, k, v, v_lr, b, s = layers[l]
            for a in range(A):
                want = orc.gqa_attention(q[a], k, v, v_lr, b[a], s, L - 1, n_q, n_kv)
                assert orc.max_rel_error(out[l, a][None, :], want) <= tol, (policy, l, a, ctx.last_kernel())
    ctx.set_kernel_policy(0)
    pool.close()


@pytest.mark.parametrize("L,P", [(1, 16), (63, 16), (64, 64), (65, 64), (777, 64), (1000, 128)])
def test_ragged_lengths_and_page_sizes(ctx, orc, L, P):
    """Partially filled last pages, single-token caches, several page sizes (fp32 pages)."""
    from paper_2602_01053_b200 import abi
    n_q, n_kv, d, r, A = 8, 2, 32, 4, 3
    pool, ad, layers = build_pool(ctx, orc, "BaseLRShared", abi.F32, 7, L, 1, n_q, n_kv, d, r, A, P=P)
    q, k, v, v_lr, b, s = layers[0]
    out = pool.decode(ad, 0, 1, [2, 0, 1, 1], n_q, np.stack([q[2][0], q[0][0], q[1][0], q[1][0]])[None])
    for i, a in enumerate([2, 0, 1, 1]):
        want = orc.gqa_attention(q[a], k, v, v_lr, b[a], s, L - 1, n_q, n_kv)
        assert orc.max_rel_error(out[0, i][None, :], want) <= 1e-4
    assert np.array_equal(out[0, 2], out[0, 3])
    pool.close()


def test_lr_append_project_matches_matmul(ctx, orc):
    """engine.hpp:414-418: V_lr rows = X * A, unscaled, computed on the device into LR pages."""
    from paper_2602_01053_b200 import abi
    L, d_model, r = 300, 192, 16
    pool, ad, layers = build_pool(ctx, orc, "BaseLRShared", abi.F32, 3, L, 1, 4, 2, 32, r, 2, d_model=d_model,
                                  project=True)
    want = layers[0][3]
    got = pool.lr_view(0, 0)
    assert got.shape == want.shape
    assert orc.max_rel_error(got, want) <= 1e-5
    # decode on the projected cache
    q, k, v, v_lr, b, s = layers[0]
    out = pool.decode(ad, 0, 1, [1], 4, q[1][None])
    assert orc.max_rel_error(out[0], orc.gqa_attention(q[1], k, v, v_lr, b[1], s, L - 1, 4, 2)) <= 1e-4
    pool.close()


@pytest.mark.parametrize("r,L,d_model,P", [(16, 300, 192, 64), (8, 77, 64, 16), (2, 45, 128, 32), (32, 1000, 4096, 64),
                                            (64, 130, 256, 128), (24, 95, 320, 64)])
def test_lr_append_project_bf16_tensor_core_kernel(ctx, orc, r, L, d_model, P):
    """bf16 pools compute V_lr = X * A (engine.hpp:414-418) with mma.sync (X rounded to bf16 as the cache dtype
    implies, A kept to fp32 accuracy by a hi + lo split) and store bf16 into the swizzled LR pages.  Checked
    against matmul (matrix.hpp:101-111) of the rounded X and the caller's un-rounded A, for every rank padding,
    ragged row counts, an append that starts mid-page and against the CUDA-core kernel (policy 1)."""
    from paper_2602_01053_b200 import Adapters, Pool, abi
    x = orc.round_bf16(orc.gaussian(L, d_model, orc.child(900 + r, 1), 1.0, np.float32))
    A = orc.gaussian(d_model, r, orc.child(900 + r, 2), 1.0 / np.sqrt(d_model), np.float32)     # NOT bf16-representable
    want = orc.matmul(x, A)
    got = {}
    for policy in (0, 1):
        ctx.set_kernel_policy(policy)
        pool = Pool(ctx, "BaseLRShared", 1, 2, 32, d_model, r, 2, max_tokens=L + 8, dtype=abi.BF16, page_tokens=P)
        ad = Adapters(ctx, 1, 2, d_model, r, 2, 32, dtype=abi.BF16)
        ad.set_a(0, A)
        pool.append_tokens(L)
        first = min(L, 37)
        assert pool.append_lr_project(ad, 0, 0, 0, x[:first]) == first
        assert pool.append_lr_project(ad, 0, 0, first, x[first:]) == L - first      # starts mid-page
        assert pool.append_lr_project(ad, 0, 0, 0, x) == 0                          # first writer wins
        got[policy] = pool.lr_view(0, 0)
        assert got[policy].shape == want.shape
        # bf16 storage: half an ulp of bf16 (2^-9) on each element, relative to the largest one
        assert orc.max_rel_error(got[policy], want) <= 4e-3, policy
        pool.close(); ad.close()
    ctx.set_kernel_policy(0)
    # same products, fp32 accumulation in a different order: the two kernels may differ by one bf16 rounding flip
    assert orc.max_rel_error(got[0], got[1]) <= 4e-3
    assert np.mean(got[0] == got[1]) > 0.98


@pytest.mark.parametrize("dtype_name,tol", [("F32", 1e-4), ("BF16", 2e-2)])
def test_prefill_block_matches_reference_path(ctx, orc, dtype_name, tol):
    """Append-step attention: L_c new rows at query_offset = L_p on a cache that already holds them
    (engine.hpp:395-443), causal rule attention.hpp:44-46."""
    from paper_2602_01053_b200 import abi
    dtype = getattr(abi, dtype_name)
    L, L_c, n_q, n_kv, d, r, A = 333, 77, 4, 2, 64, 8, 2
    pool, ad, layers = build_pool(ctx, orc, "BaseLRShared", dtype, 99, L, 1, n_q, n_kv, d, r, A)
    _, k, v, v_lr, b, s = layers[0]
    q = orc.gaussian(L_c, n_q * d, 1234, 1.0 / np.sqrt(d), np.float32)
    if dtype == abi.BF16:
        q = orc.round_bf16(q)
    for off in (L - L_c, 100, 0):
        got = pool.prefill(ad, 0, 1, n_q, q, off)
        want = orc.gqa_attention(q, k, v, v_lr, b[1], s, off, n_q, n_kv)
        assert orc.max_rel_error(got, want) <= tol
    pool.close()


def test_rank_zero_and_per_agent_schemes(ctx, orc):
    """FullShared (r = 0) is plain attention; NonShared reads the caller's own K/V set."""
    from paper_2602_01053_b200 import LorakvError, Pool, abi
    L, n_q, n_kv, d = 200, 4, 2, 32
    q, k, v, _, _, _ = synthetic_layer(orc, 5, L, 1, n_q, n_kv, d, 0, 2)
    empty_lr, empty_b = np.zeros((L, 0), np.float32), np.zeros((0, n_kv * d), np.float32)
    fs = Pool(ctx, "FullShared", 1, n_kv, d, 64, 0, 2, max_tokens=L)
    fs.append_tokens(L); fs.append_key(0, 0, 0, k); fs.append_value(0, 0, 0, v)
    out = fs.decode(None, 0, 1, [0, 1], n_q, np.stack([q[0][0], q[1][0]])[None])
    for a in range(2):
        want = orc.gqa_attention(q[a], k, v, empty_lr, empty_b, 1.0, L - 1, n_q, n_kv)
        assert orc.max_rel_error(out[0, a][None], want) <= 1e-4
    ns = Pool(ctx, "NonShared", 1, n_kv, d, 64, 0, 2, max_tokens=L)
    ns.append_tokens(L)
    ns.append_key(0, 0, 0, k); ns.append_value(0, 0, 0, v)
    ns.append_key(0, 1, 0, k * 0.5); ns.append_value(0, 1, 0, v + 1)
    o1 = ns.decode(None, 0, 1, [1], n_q, q[1][None])
    want = orc.gqa_attention(q[1], k * 0.5, v + 1, empty_lr, empty_b, 1.0, L - 1, n_q, n_kv)
    assert orc.max_rel_error(o1[0], want) <= 1e-4
    with pytest.raises(LorakvError, match="per-agent"):
        ns.decode(None, 0, 1, [0, 1], n_q, np.stack([q[0][0], q[1][0]])[None])


def test_baseshared_agent_switch_lr_prefill(ctx, orc):
    """BaseShared (kvcache.hpp:127-130, engine.hpp:411-419): the base K/V cache is shared but every agent keeps
    its own LR cache because the down-projections differ.  When another agent takes over it projects the whole
    UNSEEN context through its own A (the "LR prefill"); K/V only get the fresh rows.  Planner
    intervals, row counts and byte accounting are bit-exact vs the oracle; attention within 2e-2 (bf16 pages)."""
    from paper_2602_01053_b200 import Adapters, Pool, abi
    n_q, n_kv, d, r, N, d_model = 8, 2, 128, 16, 2, 192
    first, extra = 100, 20
    rnd = orc.round_bf16
    g = lambda rows, cols, seed, sc: rnd(orc.gaussian(rows, cols, seed, sc, np.float32))
    k = g(first + extra, n_kv * d, 1, 1.0 / np.sqrt(d)); v = g(first + extra, n_kv * d, 2, 1.0)
    x = g(first + extra, d_model, 3, 1.0)
    A = [g(d_model, r, 10 + a, 1.0 / np.sqrt(d_model)) for a in range(N)]          # per-agent A: NOT shared
    B = [g(r, n_kv * d, 20 + a, 0.02 / np.sqrt(r)) for a in range(N)]
    pool = Pool(ctx, "BaseShared", 1, n_kv, d, d_model, r, N, max_tokens=256, dtype=abi.BF16)
    st = orc.store("BaseShared", 1, n_kv * d, d_model, r, N, np.float32)
    ad = Adapters(ctx, 1, N, d_model, r, n_kv, d, dtype=abi.BF16)
    for a in range(N):
        ad.set_a_agent(0, a, A[a]); ad.set_b(0, a, B[a], 16.0)

    # agent 0 prefills the first 100 tokens
    plan = pool.plan_step(0, first)
    assert plan == orc.plan_core("BaseShared", 0, 0, first)
    assert plan["kv_project"] == (0, first) and plan["lr_project"] == (0, first)
    pool.append_tokens(first); st.append_tokens(first)
    pool.append_key(0, 0, 0, k[:first]); pool.append_value(0, 0, 0, v[:first])
    st.append_key(0, 0, 0, k[:first]); st.append_value(0, 0, 0, v[:first])
    assert pool.append_lr_project(ad, 0, 0, 0, x[:first]) == first
    st.append_lr(0, 0, 0, orc.matmul(x[:first], A[0]))
    pool.mark_seen(0); st.mark_seen(0)

    # agent 1 takes over with 20 new tokens: K/V fresh only, LR over everything it has not seen
    plan = pool.plan_step(1, extra)
    assert plan == orc.plan_core("BaseShared", first, 0, extra)
    assert plan["kv_project"] == (first, first + extra) and plan["lr_project"] == (0, first + extra)
    pool.append_tokens(extra); st.append_tokens(extra)
    lo, hi = plan["kv_project"]
    pool.append_key(0, 1, lo, k[lo:hi]); pool.append_value(0, 1, lo, v[lo:hi])
    st.append_key(0, 1, lo, k[lo:hi]); st.append_value(0, 1, lo, v[lo:hi])
    lo, hi = plan["lr_project"]
    assert pool.append_lr_project(ad, 0, 1, lo, x[lo:hi]) == hi - lo
    v_lr1 = orc.matmul(x[lo:hi], A[1])
    st.append_lr(0, 1, lo, v_lr1)
    pool.mark_seen(1); st.mark_seen(1)

    assert pool.bytes()["lr"] * 2 == st.bytes()["lr"]            # bf16 pages vs the oracle's fp32 store
    assert pool.bytes()["key"] * 2 == st.bytes()["key"]
    assert pool.rows(abi.LR, 0, 0) == first and pool.rows(abi.LR, 0, 1) == first + extra
    assert pool.seen(0) == first and pool.seen(1) == first + extra
    assert orc.max_rel_error(pool.lr_view(0, 1), v_lr1) <= 1e-2
    # agent 1 decodes over the shared K/V and ITS low-rank cache
    L = first + extra
    q = g(1, n_q * d, 77, 1.0 / np.sqrt(d))
    out = pool.decode(ad, 0, 1, [1], n_q, q[None])
    want = orc.gqa_attention(q, k, v, v_lr1, B[1], 1.0, L - 1, n_q, n_kv)
    assert orc.max_rel_error(out[0], want) <= 2e-2
    with pytest.raises(Exception, match="per-agent"):
        pool.decode(ad, 0, 1, [0, 1], n_q, np.concatenate([q, q])[None])
    pool.close(); ad.close()


# n_q, n_kv, d, r, agents, batch, L, P, layers -- rows per kv head = len(batch) * n_q / n_kv
BASESHARED_BATCHES = [
    (8, 2, 128, 16, 3, [0, 1, 2], 300, 64, 2),           # 12 rows: one warp per worker, four entries per warp tile
    (8, 2, 128, 32, 4, [3, 0, 0, 2, 1, 1, 3, 2], 257, 32, 1),   # 32 rows: two warps per worker, repeated agents
    (32, 8, 128, 16, 3, [2, 0, 1], 130, 64, 1),          # Llama head counts
    (4, 1, 128, 64, 6, [5, 4, 3, 2, 1, 0] * 6, 200, 16, 1),     # 144 rows: two row blocks, the second one ragged
    (16, 1, 64, 8, 3, [1, 2, 0], 99, 16, 1),             # group 16: one entry per warp tile; d = 64, rank 8 padded to 16
    (2, 2, 128, 16, 5, [4, 3, 2, 1, 0], 77, 16, 1),      # group 1: sixteen entries per warp tile (five used)
]


@pytest.mark.parametrize("n_q,n_kv,d,r,N,batch,L,P,n_layers", BASESHARED_BATCHES)
def test_baseshared_batched_decode_reads_kv_once(ctx, orc, n_q, n_kv, d, r, N, batch, L, P, n_layers):
    """BaseShared (kvcache.hpp:127-130, 238-243): K / V_base are shared, every agent has its OWN V_lr cache.  A batch of
    different agents runs as ONE launch that streams K / V_base once, every entry reading its own agent's page set
    (fla_decode_tma, per-entry V_lr tiles); each entry must equal gqa_attention with that agent's V_lr and B."""
    from paper_2602_01053_b200 import Adapters, Pool, abi
    rnd = orc.round_bf16
    g = lambda rows, cols, seed, sc: rnd(orc.gaussian(rows, cols, seed, sc, np.float32))
    pool = Pool(ctx, "BaseShared", n_layers, n_kv, d, 64, r, N, max_tokens=L + 8, dtype=abi.BF16, page_tokens=P)
    ad = Adapters(ctx, n_layers, N, 64, r, n_kv, d, dtype=abi.BF16)
    pool.append_tokens(L)
    k, v, lr, B = [], [], [], []
    for l in range(n_layers):
        k.append(g(L, n_kv * d, 100 + l, 1.0 / np.sqrt(d))); v.append(g(L, n_kv * d, 200 + l, 1.0))
        pool.append_key(l, 0, 0, k[l]); pool.append_value(l, 0, 0, v[l])
        lr.append([g(L, r, 300 + 10 * l + a, 1.0) for a in range(N)])
        B.append([g(r, n_kv * d, 400 + 10 * l + a, 0.02 / np.sqrt(r)) for a in range(N)])
        for a in range(N):
            # interleave the agents' appends so that their page sets are interleaved physically
            half = L // 2
            pool.append_lr(l, a, 0, lr[l][a][:half])
        for a in reversed(range(N)):
            pool.append_lr(l, a, L // 2, lr[l][a][L // 2:])
            ad.set_b(l, a, B[l][a], 16.0)
    q = np.stack([np.stack([g(1, n_q * d, 500 + 7 * l + i, 1.0 / np.sqrt(d))[0] for i in range(len(batch))]) for l in range(n_layers)])
    launches = ctx.launch_count
    out = pool.decode(ad, 0, n_layers, batch, n_q, q)
    assert ctx.last_kernel() == "fla_decode_tma"
    assert ctx.launch_count - launches == 2                      # attention + merge: one pass over K / V for the whole batch
    for l in range(n_layers):
        for i, a in enumerate(batch):
            want = orc.gqa_attention(q[l, i][None, :], k[l], v[l], lr[l][a], B[l][a], 16.0 / r, L - 1, n_q, n_kv)
            assert orc.max_rel_error(out[l, i][None, :], want) <= 2e-2, (l, i, a)
            # and the same entry alone (the one-agent-per-call path) agrees far tighter
            alone = pool.decode(ad, l, l + 1, [a], n_q, q[l, i][None, None, :])
            assert orc.max_rel_error(out[l, i][None, :], alone[0]) <= 5e-3
    ctx.set_kernel_policy(1)
    with pytest.raises(Exception, match="per-agent"):           # the CUDA-core path has no batched kernel for it
        pool.decode(ad, 0, n_layers, batch, n_q, q)
    ctx.set_kernel_policy(0)
    pool.close(); ad.close()
