"""The C oracle against the reference's own compiled headers (oracle/_ref), bit for bit.
Skipped when oracle/_ref was never built.  CPU only."""
import numpy as np
import pytest

from tests.cases import BLOCKS, fuzz_cases, synthetic_layer


@pytest.mark.parametrize("dtype,seed", [(np.float64, 20250810), (np.float32, 20250811)])
def test_oracle_bit_exact_on_acceptance_fuzz_slice(orc, ref, dtype, seed):
    """acceptance.cpp:70-83 uses seeds 20250810/20250811 with 700 base cases; a 60-case slice."""
    for c in fuzz_cases(orc, seed, 60, 64, dtype):
        assert np.array_equal(orc.naive_attention(*c), ref.naive_attention(*c))
        for br in BLOCKS:
            for bc in BLOCKS:
                a, am, ast = orc.flash_lora_attention(*c, br, bc, want_macs=True, want_stats=True)
                b, bm, bst = ref.flash_lora_attention(*c, br, bc, want_macs=True, want_stats=True)
                assert np.array_equal(a, b) and am == bm
                assert np.array_equal(ast[0], bst[0]) and np.array_equal(ast[1], bst[1])
                assert np.array_equal(orc.expand_first_attention(*c, br, bc),
                                      ref.expand_first_attention(*c, br, bc))


def test_oracle_rng_equals_reference(orc, ref):
    for seed in (0, 1, 42, 7001, 2**64 - 1):
        assert np.array_equal(orc.u64(seed, 64), ref.u64(seed, 64))
        assert orc.child(seed, 5) == ref.child(seed, 5)
        assert np.array_equal(orc.gaussian(3, 11, seed, 0.3, np.float32), ref.gaussian(3, 11, seed, 0.3, np.float32))
        assert np.array_equal(orc.gaussian(3, 11, seed, 0.3, np.float64), ref.gaussian(3, 11, seed, 0.3, np.float64))


def test_oracle_gqa_tiny_config_equals_reference(orc, ref):
    """BASELINE.json configs[0]: 4 q / 2 kv heads, d=64, r=8, 2 agents, L=512, decode."""
    q, k, v, v_lr, b, s = synthetic_layer(orc, 42, 512, 1, 4, 2, 64, 8, 2)
    for a in range(2):
        x = orc.gqa_attention(q[a], k, v, v_lr, b[a], s, 511, 4, 2)
        y = ref.gqa_attention(q[a], k, v, v_lr, b[a], s, 511, 4, 2)
        assert np.array_equal(x, y)
        assert np.array_equal(x, ref.gqa_attention(q[a], k, v, v_lr, b[a], s, 511, 4, 2, threads=4))


def test_oracle_store_equals_reference(orc, ref):
    rng = np.random.default_rng(5)
    for scheme in ("NonShared", "FullShared", "BaseShared", "BaseLRShared"):
        so = orc.store(scheme, 2, 8, 32, 4, 3, np.float32)
        sr = ref.store(scheme, 2, 8, 32, 4, 3, np.float32)
        length = 0
        for step in range(12):
            n = int(rng.integers(1, 9)); agent = int(rng.integers(0, 3))
            for s in (so, sr):
                s.append_tokens(n)
            begin = max(0, length - int(rng.integers(0, 4)))
            rows = rng.standard_normal((length + n - begin, 8)).astype(np.float32)
            lr = rng.standard_normal((length + n - begin, 4)).astype(np.float32)
            for s in (so, sr):
                for layer in range(2):
                    kb = s.key_view(layer, agent).shape[0]
                    b0 = min(begin, kb)
                    s.append_key(layer, agent, b0, rows[b0 - begin:] if b0 >= begin else np.vstack([np.zeros((begin - b0, 8), np.float32), rows]))
                    s.append_value(layer, agent, b0, rows[b0 - begin:] if b0 >= begin else np.vstack([np.zeros((begin - b0, 8), np.float32), rows]))
                    if scheme in ("BaseShared", "BaseLRShared"):
                        lb = min(begin, s.lr_view(layer, agent).shape[0])
                        s.append_lr(layer, agent, lb, lr[lb - begin:] if lb >= begin else np.vstack([np.zeros((begin - lb, 4), np.float32), lr]))
                s.mark_seen(agent)
            length += n
            assert so.bytes() == sr.bytes() and so.allocated_elements() == sr.allocated_elements()
            for layer in range(2):
                for a in range(3):
                    assert np.array_equal(so.key_view(layer, a), sr.key_view(layer, a))
                    assert np.array_equal(so.value_view(layer, a), sr.value_view(layer, a))
                    assert np.array_equal(so.lr_view(layer, a), sr.lr_view(layer, a))
                    assert so.seen(a) == sr.seen(a)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_oracle_rope_equals_reference(orc, ref, dtype):
    """detail::apply_rope (engine.hpp:225-243): the restatement is bit-identical to the reference's own code,
    including positions far into a 128K trajectory."""
    for n_heads, d_head, rows, pos in [(2, 64, 5, 0), (8, 128, 3, 131000), (1, 8, 7, 12345), (3, 6, 4, 1)]:
        m = orc.gaussian(rows, n_heads * d_head, 77 + rows, 1.0, dtype)
        a, b = orc.apply_rope(m, n_heads, d_head, pos), ref.apply_rope(m, n_heads, d_head, pos)
        assert np.array_equal(a, b)
        assert not np.array_equal(a, m) or pos == 0 and rows == 1
