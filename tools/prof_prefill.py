"""Profiling driver: the cfg3 prefill (L_c = 16K rows appended onto a 16K prefix, Llama-3.1-8B shape) on ONE
layer, a few launches of fla_prefill_umma and nothing else.  Meant to be run under ncu:

    ncu --set full --clock-control none --import-source on -k regex:fla_prefill_umma -s 2 -c 1 \
        -o gpurun_out/prefill python tools/prof_prefill.py

Without ncu it prints the CUDA-event time per launch and the achieved TFLOP/s.
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--L", type=int, default=32768)
    ap.add_argument("--Lc", type=int, default=16384)
    ap.add_argument("--rank", type=int, default=16)
    ap.add_argument("--d", type=int, default=128)
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--dtype", default="bf16", choices=["bf16", "f32"], help="f32: fp32 pages -> fla_prefill_split (bf16 planes on tcgen05)")
    args = ap.parse_args()
    import torch
    import paper_2602_01053_b200 as pkg
    from paper_2602_01053_b200 import abi

    n_q, n_kv, d, r, L, L_c, d_model = 32, 8, args.d, args.rank, args.L, args.Lc, 4096
    dt = abi.BF16 if args.dtype == "bf16" else abi.F32
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    ctx = pkg.Context(0, stream=stream.cuda_stream)
    pool = pkg.Pool(ctx, "BaseLRShared", 1, n_kv, d, d_model, r, 1, max_tokens=L, dtype=dt)
    ad = pkg.Adapters(ctx, 1, 1, d_model, r, n_kv, d, dtype=dt)
    gen = torch.Generator(device=dev)
    gen.manual_seed(1000)
    sc = float(1.0 / np.sqrt(d))
    pool.append_tokens(L)
    for c0 in range(0, L, 8192):
        n = min(8192, L - c0)
        kbuf = torch.randn((n, n_kv * d), generator=gen, device=dev, dtype=torch.float32) * sc
        vbuf = torch.randn((n, n_kv * d), generator=gen, device=dev, dtype=torch.float32)
        lbuf = torch.randn((n, max(r, 1)), generator=gen, device=dev, dtype=torch.float32)
        pool.append_device(abi.KEY, 0, 0, c0, kbuf.data_ptr(), n, n_kv * d)
        pool.append_device(abi.VALUE, 0, 0, c0, vbuf.data_ptr(), n, n_kv * d)
        if r > 0:
            pool.append_device(abi.LR, 0, 0, c0, lbuf.data_ptr(), n, max(r, 1))
    b = (np.random.default_rng(7).standard_normal((r, n_kv * d)).astype(np.float32) * (0.02 / np.sqrt(max(r, 1))))
    if r > 0:
        ad.set_b(0, 0, torch.from_numpy(b).to(torch.bfloat16).to(torch.float32).numpy(), 16.0)
    off = L - L_c
    q = (torch.randn((L_c, n_q * d), generator=gen, device=dev, dtype=torch.float32) * sc).to(torch.bfloat16).to(torch.float32)
    out = torch.empty_like(q)
    for _ in range(2):
        pool.prefill_device(ad, 0, 0, n_q, q.data_ptr(), L_c, off, out.data_ptr())
    ev0, ev1 = ctx.event(), ctx.event()
    ev0.record()
    for _ in range(args.iters):
        pool.prefill_device(ad, 0, 0, n_q, q.data_ptr(), L_c, off, out.data_ptr())
    ev1.record()
    ms = ev0.elapsed_ms(ev1) / args.iters
    pairs = L_c * off + L_c * (L_c + 1) // 2
    flops = 2 * n_q * pairs * (2 * d + r) + 2 * n_q * L_c * r * d
    print(f"{ctx.last_kernel()} L={L} L_c={L_c} r={r}: {ms:.3f} ms  {flops / ms / 1e9:.1f} TFLOP/s")


if __name__ == "__main__":
    main()
