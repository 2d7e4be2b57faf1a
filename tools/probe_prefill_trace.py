"""Per-tile clock stamps of ONE CTA of the bf16 tensor-core prefill (debug build: make EXTRA=-DLK_PREFILL_TRACE, loaded through
LORAKV_B200_LIB): when the MMA thread issued S and P V of every 64-key tile and when the two softmax warpgroups reached each
phase.  Prints the steady-state phase lengths in SM clocks.  usage: probe_prefill_trace.py [L] [L_c]"""
import ctypes as C
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2602_01053_b200 as pkg  # noqa: E402
from paper_2602_01053_b200 import abi  # noqa: E402


def main():
    L = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
    L_c = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
    n_q, n_kv, d, r, d_model = 32, 8, 128, 16, 4096
    dev = torch.device("cuda", 0)
    ctx = pkg.Context(0)
    pool = pkg.Pool(ctx, "BaseLRShared", 1, n_kv, d, d_model, r, 1, max_tokens=L, dtype=abi.BF16)
    ad = pkg.Adapters(ctx, 1, 1, d_model, r, n_kv, d, dtype=abi.BF16)
    gen = torch.Generator(device=dev); gen.manual_seed(3)
    pool.append_tokens(L)
    for c0 in range(0, L, 8192):
        n = min(8192, L - c0)
        pool.append_device(abi.KEY, 0, 0, c0, (torch.randn((n, n_kv * d), generator=gen, device=dev) * d ** -0.5).data_ptr(), n, n_kv * d)
        pool.append_device(abi.VALUE, 0, 0, c0, torch.randn((n, n_kv * d), generator=gen, device=dev).data_ptr(), n, n_kv * d)
        pool.append_device(abi.LR, 0, 0, c0, torch.randn((n, r), generator=gen, device=dev).data_ptr(), n, r)
    ad.set_b(0, 0, np.full((r, n_kv * d), 0.01, np.float32), 16.0)
    q = torch.randn((L_c, n_q * d), generator=gen, device=dev) * d ** -0.5
    out = torch.empty_like(q)
    for _ in range(3):
        pool.prefill_device(ad, 0, 0, n_q, q.data_ptr(), L_c, L - L_c, out.data_ptr())
    ctx.synchronize()
    buf = (C.c_longlong * (2048 * 16))()
    assert ctx.lib.lorakv_debug_prefill_trace(buf, 2048 * 16) == 0
    t = np.frombuffer(buf, dtype=np.int64).reshape(2048, 16).astype(np.int64)
    n = int((t[:, 6] > 0).sum())
    t = t[:n]
    t0 = t[0, 0]
    print(f"traced CTA: {n} tiles, {(t[n - 1, 6] - t0)} clocks from the first S issue to the last P = {(t[n - 1, 6] - t0) / n:.0f} per tile")
    names = ["S issued", "PV issued", "S seen", "max done", "partner max seen", "exp done", "P published"]
    lo, hi = n // 4, 3 * n // 4          # steady state
    seg = t[lo:hi]
    print(f"steady state (tiles {lo}..{hi}): period per tile {np.median(np.diff(t[lo:hi, 6])):.0f} (median of P-published differences), "
          f"{(t[hi, 6] - t[lo, 6]) / (hi - lo):.0f} mean")
    print("  per tile, relative to its own S-seen stamp (median clocks):")
    for a, b in ((2, 3), (3, 4), (4, 5), (5, 6)):
        print(f"    {names[a - 0]:>18s} -> {names[b]:<18s} {np.median(seg[:, b] - seg[:, a]):7.0f}")
    print(f"    S issued -> S seen            {np.median(seg[:, 2] - seg[:, 0]):7.0f}   (chain of 8 MMAs N=128 + look-ahead slack)")
    print(f"    P published -> PV issued      {np.median(seg[:, 1] - seg[:, 6]):7.0f}   (negative: the MMA thread was already waiting)")
    # how long a warpgroup idles between publishing P(j) and seeing S(j + 2)
    same = seg[2:, 2] - seg[:-2, 6]
    print(f"    P published(j) -> S seen(j+2) {np.median(same):7.0f}   (idle of a warpgroup between its tiles; 0 = S was waiting)")
    print("  MMA thread per tile: PV stamp, +MMAs issued, +commits issued | S stamp (even tiles), +MMAs issued")
    for j in range(lo, lo + 8):
        pv = f"PV {int(t[j, 1] - t[lo, 0])}" + (f" +{int(t[j, 8] - t[j, 1])} +{int(t[j, 9] - t[j, 8])}" if t[j, 8] > 0 else " (issued with its neighbour)")
        print(f"   tile {j}: {pv}" + (f" | S {int(t[j, 0] - t[lo, 0])} +{int(t[j, 10] - t[j, 0])}" if j % 2 == 0 else ""))
    for j in range(lo, lo + 8):
        print("   tile", j, " ".join(f"{int(t[j, s] - t[lo, 0]):7d}" for s in range(7)))
    c = np.frombuffer(buf, dtype=np.int64).reshape(2048, 16)[2047].astype(np.int64)
    first_s, first_p, last_p = t[0, 0], t[0, 6], t[n - 1, 6]
    print("  the CTA as a whole (clocks from entry): set-up done", c[1] - c[0], "| predecessor complete", c[2] - c[0], "| Q in TMEM", c[3] - c[0],
          "| first S issued", first_s - c[0], "| first P published", first_p - c[0], "| last P published", last_p - c[0],
          "| last P V complete", c[4] - c[0], "| B staged", c[5] - c[0], "| rows stored", c[6] - c[0], "| exit", c[7] - c[0])
    pool.close(); ad.close(); ctx.close()


if __name__ == "__main__":
    main()
