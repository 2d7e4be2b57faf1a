"""Decode step of one rank's kv-head shard under the cache-sharing schemes (BASELINE configs[4]: "128K shared context,
16 agents, rank 32, full 32-layer attention sweep on 8 x B200 vs non-shared and fully-shared baselines"; SURVEY 8(d)
row cfg 5).  The path shards by kv head with no communication inside attention, so what ONE of the G GPUs does is
measured exactly on one B200: rank 0's shard (n_kv / G kv heads, all layers, all agents) is built and timed here.

    python tools/scheme_compare.py [--workload cfg5] [--shard-of 8] [--steps 20] [--out gpurun_out/schemes.json]

Schemes (proj/include/lorakv/kvcache.hpp:15-21, Tables 3/4):
  BaseLRShared : one K/V_base cache + one rank-r V_lr cache for all agents, ONE batched launch per step
  FullShared   : one K/V cache, no adapter term (r = 0) -- the accuracy-losing lower bound on bytes
  BaseShared   : shared K/V_base, one V_lr cache per agent  -> ONE batched launch (every entry reads its own agent's V_lr
                 page set); "BaseShared:per-agent" times the one-launch-per-agent alternative
  NonShared    : private K/V per agent (values carry the adapter), the multi-LoRA status quo -> one launch per agent
Times are device times (events on the library's stream) of a whole step = all agents x all layers."""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import WORKLOADS, load_peaks  # noqa: E402


def run_scheme(torch, pkg, abi, ctx, scheme, wl, G, steps, warmup, per_agent_launches=False):
    desc, n_layers, n_q, n_kv, d, r, A, L, d_model = wl
    dev = torch.device("cuda", 0)
    n_kv_local = n_kv // G
    g = n_q // n_kv
    n_q_local = n_kv_local * g
    rank = r if scheme in ("BaseLRShared", "BaseShared") else 0
    pool = pkg.Pool(ctx, scheme, n_layers, n_kv, d, d_model, rank, A, max_tokens=L, dtype=abi.BF16, kv_head_begin=0, n_kv_local=n_kv_local)
    ad = pkg.Adapters(ctx, n_layers, A, d_model, rank, n_kv, d, kv_head_begin=0, n_kv_local=n_kv_local, dtype=abi.BF16) if rank else None
    gen = torch.Generator(device=dev); gen.manual_seed(5)
    chunk = 8192
    kbuf = torch.randn((chunk, n_kv * d), generator=gen, device=dev) * float(1.0 / np.sqrt(d))
    vbuf = torch.randn((chunk, n_kv * d), generator=gen, device=dev)
    lbuf = torch.randn((chunk, max(rank, 1)), generator=gen, device=dev)
    pool.append_tokens(L)
    kv_sets = range(A) if scheme == "NonShared" else (0,)
    lr_sets = range(A) if scheme == "BaseShared" else ((0,) if scheme == "BaseLRShared" else ())
    for layer in range(n_layers):
        for c0 in range(0, L, chunk):
            n = min(chunk, L - c0)
            for a in kv_sets:
                pool.append_device(abi.KEY, layer, a, c0, kbuf.data_ptr(), n, n_kv * d)
                pool.append_device(abi.VALUE, layer, a, c0, vbuf.data_ptr(), n, n_kv * d)
            for a in lr_sets:
                pool.append_device(abi.LR, layer, a, c0, lbuf.data_ptr(), n, max(rank, 1))
    torch.cuda.synchronize()
    if ad is not None:
        rng = np.random.default_rng(3)
        b = (rng.standard_normal((rank, n_kv * d)) * 0.02 / np.sqrt(rank)).astype(np.float32)
        for layer in range(n_layers):
            for a in range(A):
                ad.set_b(layer, a, b, 16.0)
    # BaseShared batches run as one launch too: K / V_base streamed once, every entry reading its own agent's V_lr set
    batched = scheme in ("BaseLRShared", "FullShared") or (scheme == "BaseShared" and not per_agent_launches)
    q = torch.randn((n_layers, A, n_q_local * d), generator=gen, device=dev) * float(1.0 / np.sqrt(d))
    out = torch.zeros_like(q)
    q_agent = [q[:, a:a + 1].contiguous() for a in range(A)]
    out_agent = [torch.zeros_like(x) for x in q_agent]

    def step():
        if batched:
            pool.decode_device(ad, 0, n_layers, list(range(A)), n_q, q.data_ptr(), out.data_ptr())
        else:       # per-agent caches serve one agent per launch (api.cu: lorakv_fla_decode_batched)
            for a in range(A):
                pool.decode_device(ad, 0, n_layers, [a], n_q, q_agent[a].data_ptr(), out_agent[a].data_ptr())

    for _ in range(warmup):
        step()
    ctx.synchronize()
    e0, e1 = ctx.event(), ctx.event()
    l0 = ctx.launch_count
    e0.record()
    for _ in range(steps):
        step()
    e1.record()
    ms = e0.elapsed_ms(e1) / steps
    launches = (ctx.launch_count - l0) // steps
    e = 2
    kv_reads = A if scheme in ("NonShared",) else (1 if batched else A)     # how often a step streams a K/V shard
    lr_reads = {"BaseLRShared": 1, "BaseShared": A}.get(scheme, 0)
    step_bytes = n_layers * (kv_reads * 2 * L * n_kv_local * d * e + lr_reads * L * rank * e)
    cb = pool.bytes()
    key_b, val_b, lr_b = cb["key"], cb["value"], cb["lr"]
    res = {"scheme": scheme + (" (one launch per agent)" if scheme == "BaseShared" and per_agent_launches else ""), "ms_per_step": ms, "agent_tok_s": A / (ms * 1e-3), "launches_per_step": int(launches),
           "kernel": ctx.last_kernel(), "streamed_bytes_per_step": int(step_bytes), "achieved_gbs": step_bytes / (ms * 1e-3) / 1e9,
           "cache_bytes": {"key": int(key_b), "value": int(val_b), "lr": int(lr_b)},
           "cache_gb": (key_b + val_b + lr_b) / 1e9, "reserved_hbm_gb": pool.reserved_bytes() / 1e9}
    pool.close()
    if ad is not None:
        ad.close()
    del kbuf, vbuf, lbuf
    torch.cuda.empty_cache()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg5", choices=sorted(WORKLOADS))
    ap.add_argument("--shard-of", type=int, default=8, help="G: time rank 0's shard of a G-GPU run")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--schemes", default="BaseLRShared,FullShared,BaseShared,BaseShared:per-agent,NonShared")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "schemes.json"))
    args = ap.parse_args()
    import torch
    import paper_2602_01053_b200 as pkg
    from paper_2602_01053_b200 import abi
    wl = WORKLOADS[args.workload]
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = pkg.Context(0, stream=stream.cuda_stream)
    peak, peak_src = load_peaks()
    rows = []
    for scheme in args.schemes.split(","):
        per_agent = scheme.endswith(":per-agent")
        res = run_scheme(torch, pkg, abi, ctx, scheme.split(":")[0], wl, args.shard_of, args.steps, args.warmup, per_agent)
        res["frac_of_hbm_peak"] = res["achieved_gbs"] / peak
        rows.append(res)
        print(json.dumps(res), flush=True)
    base = next((x for x in rows if x["scheme"] == "BaseLRShared"), rows[0])
    doc = {"workload": args.workload, "description": wl[0], "shard": f"rank 0 of {args.shard_of} (kv heads [0, {wl[3] // args.shard_of}))",
           "hbm_peak_gbs": peak, "peak_source": peak_src, "steps": args.steps, "schemes": rows}
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(doc, f, indent=1)
    md = [f"# Decode step per GPU under the cache-sharing schemes: {args.workload}, rank 0's shard of {args.shard_of} GPUs", "",
          wl[0], "",
          "| scheme | launches / step | cache on this GPU (GB) | streamed / step (GB) | ms / step | agent-tok/s | GB/s (frac of measured HBM peak) | vs BaseLRShared |",
          "|---|---|---|---|---|---|---|---|"]
    for x in rows:
        md.append(f"| {x['scheme']} | {x['launches_per_step']} | {x['cache_gb']:.2f} | {x['streamed_bytes_per_step'] / 1e9:.2f} | "
                  f"{x['ms_per_step']:.3f} | {x['agent_tok_s']:.0f} | {x['achieved_gbs']:.0f} ({x['frac_of_hbm_peak']:.2f}) | "
                  f"{x['ms_per_step'] / base['ms_per_step']:.2f}x time |")
    with open(os.path.splitext(args.out)[0] + ".md", "w") as f:
        f.write("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main()
