"""BASELINE-size parity for the two configurations whose kernels the cfg-2 test does not reach (SURVEY 8(d) "parity at scale"):

  cfg 4  Mistral-7B shape, rank 64, 8 agents sharing one 64K trajectory: 32 query rows per kv head -> the streaming kernel's
         two-warp workers; with six layers and the planning L2 shrunk to 64 MB the launch takes the in-kernel LAYER-CHUNK path
         (three chunks of two layers) that the real cfg-4 step takes at 32 layers.
  cfg 5  128K shared context, 16 agents, rank 32: 64 query rows per kv head -> the tcgen05 kernel in decode mode
         (fla_decode_umma), and -- policy 2 -- the streaming kernel's four-warp workers on the same cache.

The caches are generated on the device (as bench.py does), the sampled layers are read back through the views, and a
seeded sample of (layer, agent, kv head) triples is compared with the reference CPU path (gqa_attention over that head's
slice, attention.hpp:332-363): <= 2e-2 on max_rel_error (bf16 pages).  Needs a B200 (0.6-1.7 GB of HBM)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

N_Q, N_KV, D, D_MODEL = 32, 8, 128, 4096
G = N_Q // N_KV


@pytest.fixture(scope="module")
def ctx():
    from paper_2602_01053_b200 import Context
    c = Context(0)
    yield c
    c.close()


def build(ctx, n_layers, L, r, A, seed):
    import torch
    from paper_2602_01053_b200 import Adapters, Pool, abi
    dev = torch.device("cuda", 0)
    pool = Pool(ctx, "BaseLRShared", n_layers, N_KV, D, D_MODEL, r, A, max_tokens=L, dtype=abi.BF16)
    ad = Adapters(ctx, n_layers, A, D_MODEL, r, N_KV, D, dtype=abi.BF16)
    pool.append_tokens(L)
    gen = torch.Generator(device=dev)
    sc = float(1.0 / np.sqrt(D))
    for layer in range(n_layers):
        gen.manual_seed(seed + layer)
        for c0 in range(0, L, 8192):
            n = min(8192, L - c0)
            kbuf = torch.randn((n, N_KV * D), generator=gen, device=dev) * sc
            vbuf = torch.randn((n, N_KV * D), generator=gen, device=dev)
            lbuf = torch.randn((n, r), generator=gen, device=dev)
            pool.append_device(abi.KEY, layer, 0, c0, kbuf.data_ptr(), n, N_KV * D)
            pool.append_device(abi.VALUE, layer, 0, c0, vbuf.data_ptr(), n, N_KV * D)
            pool.append_device(abi.LR, layer, 0, c0, lbuf.data_ptr(), n, r)
        torch.cuda.synchronize()
    rng = np.random.default_rng(seed)
    rnd = lambda x: torch.from_numpy(x).to(torch.bfloat16).to(torch.float32).numpy()
    b = [[rnd((rng.standard_normal((r, N_KV * D)) * (0.02 / np.sqrt(r))).astype(np.float32)) for _ in range(A)] for _ in range(n_layers)]
    for layer in range(n_layers):
        for a in range(A):
            ad.set_b(layer, a, b[layer][a], 16.0)
    q = rnd((rng.standard_normal((n_layers, A, N_Q * D)) * sc).astype(np.float32))
    return pool, ad, q, b


def check_samples(orc, pool, out, q, b, r, L, samples):
    views = {}
    for layer, agent, kvh in samples:
        if layer not in views:
            views.clear()                                        # one layer's host copy at a time (268 / 537 MB each)
            views[layer] = (pool.key_view(layer, 0), pool.value_view(layer, 0), pool.lr_view(layer, 0))
        k, v, lr = views[layer]
        cols = slice(kvh * D, (kvh + 1) * D)
        qcols = slice(kvh * G * D, (kvh + 1) * G * D)
        want = orc.gqa_attention(np.ascontiguousarray(q[layer, agent][None, qcols]), np.ascontiguousarray(k[:, cols]),
                                 np.ascontiguousarray(v[:, cols]), lr, np.ascontiguousarray(b[layer][agent][:, cols]),
                                 16.0 / r, L - 1, G, 1)
        err = orc.max_rel_error(out[layer, agent][None, qcols], want)
        assert err <= 2e-2, (layer, agent, kvh, err)


def test_cfg4_shape_takes_the_layer_chunk_path_and_matches_the_reference(ctx, orc):
    n_layers, L, r, A = 6, 65536, 64, 8
    pool, ad, q, b = build(ctx, n_layers, L, r, A, 4400)
    agents = list(range(A))
    whole = pool.decode(ad, 0, n_layers, agents, N_Q, q)
    assert ctx.last_kernel() == "fla_decode_tma"                 # 50 MB of V_lr fit the real L2 budget: one chunk
    ctx.set_l2_bytes(64 << 20)
    try:
        out = pool.decode(ad, 0, n_layers, agents, N_Q, q)
        assert ctx.last_kernel() == "fla_decode_tma (layer chunks)"
    finally:
        ctx.set_l2_bytes(126 << 20)
    assert orc.max_rel_error(out.reshape(1, -1), whole.reshape(1, -1)) <= 5e-3        # same numbers up to the split points
    # first / last layer of a chunk, first / last agent, different kv heads
    check_samples(orc, pool, out, q, b, r, L, [(0, 0, 0), (0, 7, 5), (1, 3, 2), (5, 7, 7), (5, 0, 4)])
    # the engine-realistic call of the same shape: one layer per launch (more partials per row, the one-round-trip merge)
    one = pool.decode(ad, 3, 4, agents, N_Q, q[3:4])
    check_samples(orc, pool, np.concatenate([out[:3], one, out[4:]]), q, b, r, L, [(3, 1, 1), (3, 6, 6)])
    pool.close(); ad.close()


def test_cfg5_shape_on_the_tcgen05_decode_and_on_the_streaming_kernel(ctx, orc):
    n_layers, L, r, A = 1, 131072, 32, 16
    pool, ad, q, b = build(ctx, n_layers, L, r, A, 5500)
    agents = list(range(A))
    out = pool.decode(ad, 0, 1, agents, N_Q, q)
    assert ctx.last_kernel() == "fla_decode_umma"
    samples = [(0, 0, 0), (0, 15, 7), (0, 9, 3)]
    check_samples(orc, pool, out, q, b, r, L, samples)
    ctx.set_kernel_policy(2)                                     # keep the mma.sync streaming kernel (four-warp workers)
    try:
        out2 = pool.decode(ad, 0, 1, agents, N_Q, q)
        assert ctx.last_kernel().startswith("fla_decode_tma")
    finally:
        ctx.set_kernel_policy(0)
    check_samples(orc, pool, out2, q, b, r, L, [(0, 4, 6)])
    assert orc.max_rel_error(out2.reshape(1, -1), out.reshape(1, -1)) <= 5e-3
    pool.close(); ad.close()
