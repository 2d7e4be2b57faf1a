"""Fixed cost of ONE decode launch per layer (the engine-realistic call: layer l+1's q depends on layer l).

For a cfg-2-shaped pool (32q / 8kv, d 128, rank 16, 3 agents) of n_layers layers it times, per context length L:
  * a run of per-layer decode calls issued back to back (device time per call, events on the library's stream),
  * the attention kernel alone (lorakv_ctx_mean_kernel_ms),
and fits  t(L) = a + bytes(L) / bw.  Usage: python tools/probe_layer_launch.py [n_layers] [reps]"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2602_01053_b200 as pkg  # noqa: E402
from paper_2602_01053_b200 import abi  # noqa: E402


def main():
    n_layers = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    n_q, n_kv, d, r, A, d_model = 32, 8, 128, 16, 3, 4096
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    ctx = pkg.Context(0, stream=stream.cuda_stream)
    Ls = [int(x) for x in os.environ.get("PROBE_LS", "1024,4096,8192,16384,32768,65536").split(",")]
    Lmax = max(Ls)
    rows = []
    for L in Ls:
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
        torch.cuda.synchronize()
        q = torch.randn((n_layers, A, n_q * d), device=dev) * (d ** -0.5)
        out = torch.zeros_like(q)
        ids = list(range(A))

        def sweep():
            for layer in range(n_layers):
                pool.decode_device(ad, layer, layer + 1, ids, n_q, q[layer].data_ptr(), out[layer].data_ptr())

        for _ in range(3):
            sweep()
        ctx.synchronize()
        e0, e1 = ctx.event(), ctx.event()
        e0.record()
        for _ in range(reps):
            sweep()
        e1.record()
        per_call = e0.elapsed_ms(e1) / (reps * n_layers) * 1e3
        ctx.set_profiling(True)
        for _ in range(max(1, min(reps, 256 // n_layers))):
            sweep()
        kern, n_calls = ctx.mean_kernel_ms()
        ctx.set_profiling(False)
        nbytes = 2 * L * n_kv * d * 2 + L * r * 2 + 2 * A * n_q * d * 4 + A * r * n_kv * d * 4
        rows.append((L, nbytes, per_call, kern * 1e3))
        print(f"L={L:6d} bytes={nbytes / 1e6:8.2f} MB  per-call {per_call:7.2f} us  kernel {kern * 1e3:7.2f} us "
              f"({nbytes / (kern * 1e-3) / 1e9:7.1f} GB/s) kernel={ctx.last_kernel()}", flush=True)
        pool.close(); ad.close()
    x = np.array([r_[1] for r_ in rows], dtype=np.float64)
    for name, col in (("per-call", 2), ("kernel", 3)):
        y = np.array([r_[col] for r_ in rows], dtype=np.float64)
        b, a = np.polyfit(x, y, 1)
        print(f"fit {name}: fixed {a:6.2f} us + bytes / {1e-3 / b:7.1f} GB/s")
    ctx.close()


if __name__ == "__main__":
    main()
