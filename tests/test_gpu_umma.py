"""tcgen05 operand conventions (lorakv_selftest_umma): the shared-memory layouts that pages land in
after a bulk copy -- K-major SWIZZLE_128B for K, MN-major SWIZZLE_128B/64B/32B for V and V_lr
(csrc/page_layout.cuh) -- are exactly what the tensor cores expect, and TMEM accumulators survive a
tcgen05.ld / scale / tcgen05.st round trip (the lazy O rescale of the prefill kernel).  Needs a B200."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    from paper_2602_01053_b200 import Context
    c = Context(0)
    yield c
    c.close()


def bf16(x):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).to(torch.bfloat16).to(torch.float32).numpy()


@pytest.mark.parametrize("N,K,mn_major", [(128, 128, False), (64, 64, False), (256, 128, False), (16, 64, False),
                                          (128, 128, True), (64, 128, True), (32, 128, True), (16, 128, True),
                                          (192, 64, True), (16, 64, True)])
@pytest.mark.parametrize("rescale", [False, True])
@pytest.mark.parametrize("a_in_tmem", [False, True])
def test_umma_tile_matches_host_matmul(ctx, N, K, mn_major, rescale, a_in_tmem):
    rng = np.random.default_rng(N * 1000 + K + int(mn_major))
    a = bf16(rng.standard_normal((128, K)))
    b = bf16(rng.standard_normal((K, N) if mn_major else (N, K)))
    want = a.astype(np.float64) @ (b if mn_major else b.T).astype(np.float64)
    alpha = 0.375
    got = ctx.selftest_umma(a, b, mn_major, alpha=alpha, rescale=rescale, a_in_tmem=a_in_tmem)
    if rescale:
        want = want * (alpha + 1.0)
    err = np.abs(got - want).max() / np.abs(want).max()
    assert err <= 1e-5, (N, K, mn_major, rescale, a_in_tmem, err)


@pytest.mark.parametrize("N,K", [(128, 16), (128, 32), (64, 16), (256, 32), (16, 16)])
@pytest.mark.parametrize("rescale", [False, True])
def test_umma_narrow_k_major_rows(ctx, N, K, rescale):
    """A tile of the key-side low-rank cache L_k: [keys][rank_k] rows of 32 / 64 bytes (SWIZZLE_32B / 64B), consumed as a
    K-major B operand with A from TMEM -- the extra k block of the score product on the tcgen05 kernels."""
    rng = np.random.default_rng(77 * N + K)
    a = bf16(rng.standard_normal((128, K)))
    b = bf16(rng.standard_normal((N, K)))
    want = a.astype(np.float64) @ b.T.astype(np.float64)
    got = ctx.selftest_umma(a, b, False, alpha=0.375, rescale=rescale, a_in_tmem=True)
    if rescale:
        want = want * 1.375
    err = np.abs(got - want).max() / np.abs(want).max()
    assert err <= 1e-5, (N, K, rescale, err)
