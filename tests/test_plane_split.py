"""The arithmetic behind the fp32-mode tensor-core kernels (csrc/fla_prefill_split.cu, the plane projections in
csrc/kv_project_umma.cu, the P V step of csrc/fla_decode_f32.cu): an fp32 number is a sum of bf16 planes, exact to 2^-25 with
three planes and 2^-16 with two, and a dot product of two such sums is the sum of the pairwise plane products the tensor cores
accumulate in fp32 -- six of them reproduce the fp32 product to ~2^-24, three the 2^-16 the P V step needs.  CPU only: numpy
float64 as the referee, bf16 rounding from the checker (round-to-nearest-even, as cvt.rn.bf16x2.f32)."""
import numpy as np


def planes(orc, x, n):
    out, r = [], x.astype(np.float32).copy()
    for _ in range(n):
        p = orc.round_bf16(r)
        out.append(p)
        r = (r - p).astype(np.float32)          # exact: both are fp32 numbers within a factor 2^9 of each other
    return out


def test_bf16_planes_reconstruct_fp32(orc):
    rng = np.random.default_rng(5)
    x = (rng.standard_normal((64, 257)) * np.exp(rng.uniform(-20, 20, (64, 257)))).astype(np.float32)
    p3, p2 = planes(orc, x, 3), planes(orc, x, 2)
    err3 = np.abs(sum(p.astype(np.float64) for p in p3) - x.astype(np.float64)) / np.abs(x)
    err2 = np.abs(sum(p.astype(np.float64) for p in p2) - x.astype(np.float64)) / np.abs(x)
    assert err3.max() <= 2.0 ** -25 and err2.max() <= 2.0 ** -16
    # every plane is a bf16 number (re-rounding changes nothing) and the subtraction chain loses nothing
    for p in p3:
        assert np.array_equal(orc.round_bf16(p), p)


def test_six_plane_products_give_the_fp32_dot_product(orc):
    """scores: q.k = q0k0 + q0k1 + q1k0 + q0k2 + q2k0 + q1k1 (dropped: q1k2, q2k1, q2k2 <= 2^-25 |q||k|); amplitude 25 as in the
    reference's fuzz grid, where the scaled scores reach the hundreds and an absolute error is a relative error of exp()."""
    rng = np.random.default_rng(6)
    d = 128
    for amp in (1.0, 25.0):
        q = (rng.standard_normal((32, d)) * amp / np.sqrt(d)).astype(np.float32)
        k = (rng.standard_normal((200, d)) * amp / np.sqrt(d)).astype(np.float32)
        qp, kp = planes(orc, q, 3), planes(orc, k, 3)
        pairs = [(1, 1), (0, 2), (2, 0), (0, 1), (1, 0), (0, 0)]                     # the kernels' order: smallest terms first
        got = sum(qp[a].astype(np.float64) @ kp[b].astype(np.float64).T for a, b in pairs)
        want = q.astype(np.float64) @ k.astype(np.float64).T
        scale = 1.0 / np.sqrt(d)
        assert np.abs(got - want).max() * scale <= 2e-6 * max(1.0, amp * amp / 25.0), amp   # absolute error of the scaled score
        two = sum(qp[a].astype(np.float64) @ kp[b].astype(np.float64).T for a, b in [(0, 1), (1, 0), (0, 0)])
        if amp == 25.0:                      # two planes would eat the whole 1e-4 budget in the exponent (x log2 e: 1.4e-4)
            assert np.abs(two - want).max() * scale > 5e-5


def test_three_plane_products_are_enough_for_p_v(orc):
    """P V = p0v0 + p1v0 + p0v1 with P in [0, 1]: relative to the row's output the error stays far inside 1e-4."""
    rng = np.random.default_rng(7)
    p = rng.uniform(0, 1, (16, 4096)).astype(np.float32) ** 8        # a peaked distribution of weights
    v = rng.standard_normal((4096, 128)).astype(np.float32)
    pp, vp = planes(orc, p, 2), planes(orc, v, 2)
    got = sum(pp[a].astype(np.float64) @ vp[b].astype(np.float64) for a, b in [(1, 0), (0, 1), (0, 0)])
    want = p.astype(np.float64) @ v.astype(np.float64)
    assert np.abs(got - want).max() / np.abs(want).max() <= 1e-5
