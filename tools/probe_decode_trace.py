"""Phase timestamps of one single-layer decode launch (debug build: make EXTRA=-DLK_DECODE_TRACE, loaded through
LORAKV_B200_LIB).  Prints, over the warps of the launch, when each phase was reached relative to the first warp's entry."""
import ctypes as C
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2602_01053_b200 as pkg  # noqa: E402
from paper_2602_01053_b200 import abi  # noqa: E402

NAMES = ["entry", "barriers ready", "ring primed (producer issued)", "before first full wait", "first tile landed",
         "first tile done", "all tiles done", "partial flushed", "predecessor complete (pdl_wait)", "Q fragments packed",
         "first stage issued", "2nd issue: empty wait passed", "2nd issue: expect_tx done", "2nd issue: copies issued", "Q loads issued"]


def main():
    L = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
    n_layers = 4
    n_q, n_kv, d, r, A, d_model = 32, 8, 128, 16, 3, 4096
    if len(sys.argv) > 3:                      # other batch shapes: probe_decode_trace.py L agents rank (cfg 4: 65536 8 64)
        A, r = int(sys.argv[2]), int(sys.argv[3])
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    ctx = pkg.Context(0, stream=stream.cuda_stream)
    pool = pkg.Pool(ctx, "BaseLRShared", n_layers, n_kv, d, d_model, r, A, max_tokens=L, dtype=abi.BF16)
    ad = pkg.Adapters(ctx, n_layers, A, d_model, r, n_kv, d, dtype=abi.BF16)
    pool.append_tokens(L)
    gen = torch.Generator(device=dev)
    gen.manual_seed(1)
    for layer in range(n_layers):
        for c0 in range(0, L, 8192):
            n = min(8192, L - c0)
            kbuf = torch.randn((n, n_kv * d), generator=gen, device=dev) * (d ** -0.5)
            vbuf = torch.randn((n, n_kv * d), generator=gen, device=dev)
            lbuf = torch.randn((n, r), generator=gen, device=dev)
            pool.append_device(abi.KEY, layer, 0, c0, kbuf.data_ptr(), n, n_kv * d)
            pool.append_device(abi.VALUE, layer, 0, c0, vbuf.data_ptr(), n, n_kv * d)
            pool.append_device(abi.LR, layer, 0, c0, lbuf.data_ptr(), n, r)
        for a in range(A):
            ad.set_b(layer, a, np.zeros((r, n_kv * d), np.float32) + 0.01, 16.0)
    q = torch.randn((n_layers, A, n_q * d), device=dev) * (d ** -0.5)
    out = torch.zeros_like(q)
    ids = list(range(A))
    for rep in range(3):
        for layer in range(n_layers):
            pool.decode_device(ad, layer, layer + 1, ids, n_q, q[layer].data_ptr(), out[layer].data_ptr())
    ctx.synchronize()
    lib = ctx.lib
    buf = (C.c_ulonglong * (1024 * 16))()
    assert lib.lorakv_debug_decode_trace(buf, 1024 * 16) == 0
    t = np.frombuffer(buf, dtype=np.uint64).reshape(1024, 16).astype(np.int64)
    live = t[:, 0] > 0
    t = t[live]
    t0 = t[:, 0].min()
    print(f"L={L}: {live.sum()} warps traced; times in us relative to the first warp's entry (min / median / max over warps)")
    for s, name in enumerate(NAMES):
        col = (t[:, s] - t0) / 1e3
        col = col[t[:, s] > 0]
        if len(col):
            print(f"  {s} {name:32s} {col.min():7.2f} {np.median(col):7.2f} {col.max():7.2f}")
    # per-warp durations
    dur_tiles = (t[:, 6] - t[:, 4]) / 1e3
    print(f"  main loop (first tile landed -> all tiles done): min {dur_tiles.min():.2f} median {np.median(dur_tiles):.2f} max {dur_tiles.max():.2f} us")
    print(f"  first tile: median {(np.median(t[:, 5] - t[:, 4])) / 1e3:.2f} us")
    # the merge kernel of the same (last) layer-step, relative to the same origin
    mbuf = (C.c_ulonglong * (512 * 4))()
    if hasattr(lib, "lorakv_debug_merge_trace") and lib.lorakv_debug_merge_trace(mbuf, 512 * 4) == 0:
        m = np.frombuffer(mbuf, dtype=np.uint64).reshape(512, 4).astype(np.int64)
        m = m[m[:, 0] > 0]
        for s_, name in enumerate(["merge CTA entry", "merge set up (before the wait)", "merge wait returned", "merge row stored"]):
            col = (m[:, s_] - t0) / 1e3
            print(f"  M{s_} {name:31s} {col.min():7.2f} {np.median(col):7.2f} {col.max():7.2f}")
    pool.close(); ad.close()
    ctx.close()


if __name__ == "__main__":
    main()
