"""Seeded input builders shared by the parity tests.  They restate how the reference's own tests
build inputs (tests/test_attention.cpp:32-43 random_case, include/lorakv/fuzz.hpp:33-46)."""
import numpy as np


def random_case(chk, L, L_c, d, r, offset, seed, dtype):
    """tests/test_attention.cpp:32-43: q,k,v,v_lr,b_up ~ N(0,1) from Rng(seed).child(1..5)."""
    g = lambda rows, cols, key: chk.gaussian(rows, cols, chk.child(seed, key), 1.0, dtype)
    return [g(L_c, d, 1), g(L, d, 2), g(L, d, 3), g(L, r, 4), g(r, d, 5), 0.5, offset]


def fuzz_cases(chk, seed, n_cases, max_len, dtype):
    """include/lorakv/fuzz.hpp:25-55: shapes and amplitudes of run_kernel_fuzz."""
    root = chk.mix(seed, 0xF022)
    for c in range(n_cases):
        s = chk.child(root, c)
        u = chk.u64(s, 6)
        L = 1 + int(u[0] % np.uint64(max_len))
        L_c = 1 + int(u[1] % np.uint64(L))
        off = int(u[2] % np.uint64(L - L_c + 1))
        r = [0, 1, 2, 8][int(u[3] % np.uint64(4))]
        d = [4, 16, 64][int(u[4] % np.uint64(3))]
        amp = [1.0, 5.0, 25.0][int(u[5] % np.uint64(3))]
        g = lambda rows, cols, key, sc: chk.gaussian(rows, cols, chk.child(s, key), sc, dtype)
        sc = amp / np.sqrt(float(d))
        yield [g(L_c, d, 1, sc), g(L, d, 2, sc), g(L, d, 3, 1.0), g(L, r, 4, 1.0), g(r, d, 5, 1.0),
               0.5, off]


BLOCKS = (1, 3, 8, 64)


def synthetic_layer(chk, seed, L, L_c, n_q, n_kv, d, r, n_agents, dtype=np.float32, amp=1.0):
    """SURVEY.md 8(d) synthetic inputs: Rng(seed).child(1..5) = q, k, v_base, v_lr, b_up;
    q,k ~ N(0, amp/sqrt(d)), v ~ N(0,1), b_up ~ N(0, 0.02/sqrt(r)) per agent (engine.hpp:169),
    lr_scale = 16/r (engine.hpp:124)."""
    sc = amp / np.sqrt(float(d))
    q = [chk.gaussian(L_c, n_q * d, chk.child(chk.child(seed, 1), a), sc, dtype) for a in range(n_agents)]
    k = chk.gaussian(L, n_kv * d, chk.child(seed, 2), sc, dtype)
    v = chk.gaussian(L, n_kv * d, chk.child(seed, 3), 1.0, dtype)
    v_lr = chk.gaussian(L, r, chk.child(seed, 4), 1.0, dtype)
    b = [chk.gaussian(r, n_kv * d, chk.child(chk.child(seed, 5), a), 0.02 / np.sqrt(max(r, 1)), dtype)
         for a in range(n_agents)]
    lr_scale = 16.0 / r if r > 0 else 1.0
    return q, k, v, v_lr, b, lr_scale


# ---- snapshot fixtures (kvcache.hpp:438-546): one small caught-up store per scheme, values are small integers so
# that fp32 and bf16 pools hold them exactly (the pattern of tests/test_kvcache.cpp fill_rows / fill_caught_up) ----
SNAPSHOT_DIMS = dict(n_layers=2, d_kv=16, d_model=16, rank=2, n_agents=3, n_kv_heads=2, L=9)
SNAPSHOT_SCHEMES = ["NonShared", "FullShared", "BaseShared", "BaseLRShared"]


def snapshot_rows(kind, layer, agent, L, cols):
    """kind 0 key, 1 value, 2 lr"""
    i = np.arange(L)[:, None]; j = np.arange(cols)[None, :]
    v = (i * 17 + j * 3 + 1000 * layer + 7 * agent + 50 * kind) % 251 - 100
    return v.astype(np.float32)


def snapshot_fill(store_like, scheme):
    """Drive any object with append_tokens / append_key / append_value / append_lr / mark_seen the same way."""
    d = SNAPSHOT_DIMS
    L = d["L"]
    store_like.append_tokens(L)
    kv_agents = range(d["n_agents"]) if scheme == "NonShared" else [0]
    for layer in range(d["n_layers"]):
        for a in kv_agents:
            store_like.append_key(layer, a, 0, snapshot_rows(0, layer, a, L, d["d_kv"]))
            store_like.append_value(layer, a, 0, snapshot_rows(1, layer, a, L, d["d_kv"]))
        if scheme == "BaseShared":
            for a in range(d["n_agents"]):
                store_like.append_lr(layer, a, 0, snapshot_rows(2, layer, a, L - a, d["rank"]))     # ragged LR prefills
        elif scheme == "BaseLRShared":
            store_like.append_lr(layer, 0, 0, snapshot_rows(2, layer, 0, L, d["rank"]))
    store_like.mark_seen(0)
    store_like.mark_seen(2)
