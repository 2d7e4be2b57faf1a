#!/usr/bin/env python
"""bench.py -- Flash-LoRA-Attention batched decode on B200 (BASELINE.json metric).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--workload cfg2|cfg1|cfg4|cfg5]

One "step" = one decode step of the whole agent batch: every agent's query attends to the shared
trajectory through ALL layers of the model (32 for the Llama-3.1-8B shape), i.e. one pass of the hot
path gqa_attention (reference: proj/include/lorakv/attention.hpp:332, called per agent per layer by
engine.hpp:440-443).  Metric: agent-tokens per second (= agents / step time).

  value     inputs (paged K/V/V_lr cache, B tables, q) resident in HBM, CUDA-event timed
  e2e       the same step through the C ABI with HOST buffers: q pinned host -> device, kernels,
            output device -> host, inside the timed region (wall clock, synchronised both sides)
  roofline  dominant kernel's algorithmic bytes / its CUDA-event duration vs MEASURED_PEAKS.json
  cpu_baseline  the reference CPU path (oracle/_ref when built, else the oracle port) on the host
            cores, bounded sample (rank 0, N = 1 only)

N > 1 (torchrun, one rank per GPU): KV heads are sharded across ranks (north star: no communication
inside attention); the only collective is the end-of-step all-gather of the output slab (NCCL).
The total work is fixed, so scaling is "strong".

--impl reference times the reference's own CPU implementation of the path on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # name: (description, n_layers, n_q, n_kv, d_head, rank, agents, L, d_model)
    "cfg1": ("tiny single-layer: 4q/2kv heads, d=64, r=8, 2 agents, 512-token context, decode", 1, 4, 2, 64, 8, 2, 512, 256),
    "cfg2": ("Llama-3.1-8B attention shape (32q/8kv, d=128), r=16, 3 agents, 32K shared trajectory, batched decode", 32, 32, 8, 128, 16, 3, 32768, 4096),
    "cfg4": ("Mistral-7B shape (32q/8kv, d=128), r=64, 8 agents, 64K shared trajectory, decode", 32, 32, 8, 128, 64, 8, 65536, 4096),
    "cfg5": ("long-context stress: 128K shared context, 16 agents, r=32, 32-layer sweep", 32, 32, 8, 128, 32, 16, 131072, 4096),
}


def algorithmic_bytes(n_layers, n_q, n_kv_local, n_kv, d, r, A, L, e):
    """per layer 2*L*n_kv'*d*e [K+V] + L*r*e [V_lr] + 2*A*g*n_kv'*d*4 [q,out fp32] + A*r*n_kv'*d*4 [B]."""
    g = n_q // n_kv
    per_layer = 2 * L * n_kv_local * d * e + L * r * e + 2 * A * g * n_kv_local * d * 4 + A * r * n_kv_local * d * 4
    return n_layers * per_layer


class ClockSampler:
    """SM clocks and throttle reasons DURING the timed region (B200_PROFILING.md).  The region lasts
    milliseconds, so a thread polls NVML directly (about every millisecond) instead of parsing
    `nvidia-smi -lms`; nvidia-smi remains the fallback when the NVML binding is missing."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device, self.proc, self.path = device, None, None
        self.thread, self.stop_flag, self.samples, self.reasons = None, threading.Event(), [], set()
        self.max_mhz, self.nvml = None, None

    def _visible_index(self):
        vis = os.environ.get("CUDA_VISIBLE_DEVICES")
        if vis:
            try:
                return int(vis.split(",")[self.device])
            except Exception:
                pass
        return self.device

    def _poll(self, h):
        n = self.nvml
        bits = {"hw_slowdown": n.nvmlClocksEventReasonHwSlowdown, "hw_thermal_slowdown": n.nvmlClocksEventReasonHwThermalSlowdown,
                "sw_thermal_slowdown": n.nvmlClocksEventReasonSwThermalSlowdown, "sw_power_cap": n.nvmlClocksEventReasonSwPowerCap}
        while not self.stop_flag.is_set():
            try:
                self.samples.append(float(n.nvmlDeviceGetClockInfo(h, n.NVML_CLOCK_SM)))
                r = n.nvmlDeviceGetCurrentClocksEventReasons(h)
                for name, bit in bits.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                break
            time.sleep(0.0005)

    def start(self):
        try:
            import pynvml as n
            n.nvmlInit()
            h = n.nvmlDeviceGetHandleByIndex(self._visible_index())
            self.max_mhz = float(n.nvmlDeviceGetMaxClockInfo(h, n.NVML_CLOCK_SM))
            self.nvml = n
            self.thread = threading.Thread(target=self._poll, args=(h,), daemon=True)
            self.thread.start()
            return
        except Exception:
            self.thread = None
        try:
            f = tempfile.NamedTemporaryFile("w", suffix=".csv", delete=False)
            self.path = f.name
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-i", str(self.device), "-lms", "100"], stdout=f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        out = {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        if self.thread:
            self.stop_flag.set()
            self.thread.join(timeout=2)
            if self.samples:
                out.update(sm_mhz=statistics.median(self.samples), sm_max_mhz=self.max_mhz, reasons=sorted(self.reasons),
                           samples=len(self.samples), source="nvml")
            return out
        if not self.proc:
            return out
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        try:
            for line in open(self.path):
                p = [x.strip() for x in line.split(",")]
                if len(p) < 9:
                    continue
                try:
                    sm.append(float(p[1])); mx.append(float(p[2]))
                except ValueError:
                    continue
                for name, v in zip(("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"), p[5:9]):
                    if v.lower().startswith("active"):
                        reasons.add(name)
            os.unlink(self.path)
        except Exception:
            pass
        if sm:
            out.update(sm_mhz=statistics.median(sm), sm_max_mhz=max(mx), reasons=sorted(reasons), samples=len(sm),
                       source="nvidia-smi")
        return out


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def round_bf16_np(x):
    """float32 -> nearest bf16 (ties to even) -> float32, in numpy (both arms round the same way)."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    r = ((u >> 16) & 1) + np.uint32(0x7FFF)
    return ((u + r) & np.uint32(0xFFFF0000)).view(np.float32)


def synthetic_layer_inputs(layer, L, n_q, n_kv, d, r, A, bf16):
    """The synthetic operands of one layer, shared by the GPU arm and the reference arm so that both see the SAME numbers
    (SURVEY 8(d) scales: q, k ~ N(0, 1/sqrt(d)), v, v_lr ~ N(0, 1), b_up ~ N(0, 0.02/sqrt(r)); bf16 mode rounds every
    operand once).  Returns k, v, v_lr, [q per agent], [b_up per agent]."""
    rng = np.random.default_rng([42, layer])
    sc = np.float32(1.0 / np.sqrt(d))
    k = rng.standard_normal((L, n_kv * d), dtype=np.float32) * sc
    v = rng.standard_normal((L, n_kv * d), dtype=np.float32)
    v_lr = rng.standard_normal((L, max(r, 1)), dtype=np.float32)[:, :r]
    q = [rng.standard_normal((1, n_q * d), dtype=np.float32) * sc for _ in range(A)]
    b = [rng.standard_normal((r, n_kv * d), dtype=np.float32) * np.float32(0.02 / np.sqrt(max(r, 1))) for _ in range(A)]
    rnd = round_bf16_np if bf16 else (lambda x: np.ascontiguousarray(x, dtype=np.float32))
    return rnd(k), rnd(v), np.ascontiguousarray(rnd(v_lr)), [rnd(x) for x in q], [rnd(x) for x in b]


def cpu_reference_time(chk, q_list, k, v, v_lr, b_list, lr_scale, L, n_q, n_kv, threads):
    """One layer x all agents through the reference CPU path; returns seconds."""
    t0 = time.perf_counter()
    outs = []
    for a in range(len(q_list)):
        outs.append(chk.gqa_attention(q_list[a], k, v, v_lr, b_list[a], lr_scale, L - 1, n_q, n_kv, threads=threads))
    return time.perf_counter() - t0, outs


def run_reference(args, wl):
    """--impl reference: the reference's own CPU implementation of the path on the host cores."""
    from oracle import checker
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    desc, n_layers, n_q, n_kv, d, r, A, L, d_model = wl
    chk = checker.best()
    threads = host_threads()
    # the operands of layer 0 of the GPU arm (same generator, same seed, same bf16 rounding in bf16 mode)
    k, v, v_lr, q, b = synthetic_layer_inputs(0, L, n_q, n_kv, d, r, A, args.dtype == "bf16")
    lr_scale = 16.0 / r if r else 1.0
    # One step = the whole decode step: every layer x every agent through gqa_attention<float>.  The layers run over layer
    # 0's cache contents (the CPU path's time does not depend on the values; 32 distinct layers would need 8.6 GB of host
    # memory for nothing).  The driver's K / W decide how many whole steps are timed.
    t_first, _o = cpu_reference_time(chk, q, k, v, v_lr, b, lr_scale, L, n_q, n_kv, threads)
    for _ in range(max(args.warmup - 1, 0)):
        cpu_reference_time(chk, q, k, v, v_lr, b, lr_scale, L, n_q, n_kv, threads)      # one layer per warm-up step
    # bounded: the timed region stays within ~4 minutes; at cfg 2 that is all 32 layers of every step
    layers_timed = int(min(n_layers, max(1, 240.0 / (max(args.steps, 1) * max(t_first, 1e-3)))))

    def whole_step():
        t = 0.0
        for _ in range(layers_timed):
            s_, _o = cpu_reference_time(chk, q, k, v, v_lr, b, lr_scale, L, n_q, n_kv, threads)
            t += s_
        return t
    t0 = time.perf_counter()
    layer_s = []
    for _ in range(args.steps):
        layer_s.append(whole_step() / layers_timed)
    step_s = (time.perf_counter() - t0) / args.steps * (n_layers / layers_timed)
    per_layer = statistics.mean(layer_s)
    value = A / step_s
    # the same path on ONE host thread (BASELINE.md asks for both): one layer x one agent, scaled
    t1 = time.perf_counter()
    chk.gqa_attention(q[0], k, v, v_lr, b[0], lr_scale, L - 1, n_q, n_kv, threads=1)
    one_thread_layer_agent_s = time.perf_counter() - t1
    one_thread_value = A / (one_thread_layer_agent_s * A * n_layers)
    sample = (f"every step runs {layers_timed} of {n_layers} layers x {A} agents (gqa_attention<float>, {threads} threads over q heads; "
              f"measured {per_layer:.3f} s per layer" + ("" if layers_timed == n_layers else f", scaled by {n_layers}/{layers_timed}") +
              ") over layer 0's synthetic cache contents, the operands the GPU arm uses for that layer")
    line = {
        "impl": "reference", "metric": "flash_lora_attn_decode_agent_tokens_per_s", "value": value, "unit": "tok/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_s * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": args.workload, "description": desc, "n_layers": n_layers, "agents": A, "context": L, "rank": r,
                   "operands": "bf16-rounded values in f32 arithmetic" if args.dtype == "bf16" else "f32"},
        "cpu_baseline": {"value": value, "unit": "tok/s", "cores": threads, "kind": chk.kind, "sample": sample,
                         "seconds_per_layer": per_layer,
                         "one_thread": {"value": one_thread_value, "unit": "tok/s", "cores": 1,
                                        "sample": f"1 layer x 1 agent timed once ({one_thread_layer_agent_s:.2f} s) and scaled by {n_layers} x {A}"}},
        "e2e": {"value": value, "unit": "tok/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def load_tensor_peak():
    """(burst peak, source, sustained peak or None): the burst figure is the roofline denominator of a kernel timed
    alone; the sustained one (cuBLAS under the 1 kW power cap) is reported beside it because the prefill kernel runs at
    the cap as well (sw_power_cap active, SM clock ~1.6 GHz: profiles/r1_clocks_prefill.txt)."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["bf16_tflops"]), "measured (MEASURED_PEAKS.json bf16_tflops, burst)", p.get("bf16_tflops_sustained")
    except Exception:
        return 1590.0, "fallback (B200_PROFILING.md 1.59 PFLOP/s)", 1400.0


def bench_prefill(args, torch, ctx, pool, ad, dev, n_layers, n_q, n_kv, d, r, L, d_model):
    """TTFT of one layer: X*A projection of the L_c new rows (the V_lr append of engine.hpp:414-418, timed
    on a scratch pool so the trajectory is untouched) + Flash-LoRA-Attention of the L_c query rows at
    query_offset = L - L_c over the cached trajectory (lorakv_fla_prefill), device-resident operands."""
    import paper_2602_01053_b200 as pkg
    from paper_2602_01053_b200 import abi
    L_c = L // 2
    off = L - L_c
    gen = torch.Generator(device=dev); gen.manual_seed(77)
    sc = float(1.0 / np.sqrt(d))
    q = (torch.randn((L_c, n_q * d), generator=gen, device=dev, dtype=torch.float32) * sc).to(torch.bfloat16).to(torch.float32)
    out = torch.empty_like(q)
    steps = max(3, min(args.steps, 10))
    for _ in range(2):
        pool.prefill_device(ad, 0, 1, n_q, q.data_ptr(), L_c, off, out.data_ptr())
    ev0, ev1 = ctx.event(), ctx.event()
    sampler = ClockSampler(torch.cuda.current_device())
    torch.cuda.synchronize()
    sampler.start()
    ev0.record()
    for i in range(steps):
        pool.prefill_device(ad, i % n_layers, 1, n_q, q.data_ptr(), L_c, off, out.data_ptr())
    ev1.record()
    attn_ms = ev0.elapsed_ms(ev1) / steps
    prefill_clocks = sampler.stop()
    kernel = ctx.last_kernel()
    pairs = L_c * off + L_c * (L_c + 1) // 2
    flops = 2 * n_q * pairs * (2 * d + r) + 2 * n_q * L_c * r * d
    peak, peak_src, peak_sustained = load_tensor_peak()
    traffic = None
    try:   # DRAM bytes of one launch from the committed `ncu --set full` capture (profiles/)
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            traffic = json.load(f).get(f"cfg3_{args.dtype}_{kernel}")
    except Exception:
        pass
    res = {"workload": "cfg3", "L_c": L_c, "query_offset": off, "attention_ms_per_layer": attn_ms,
           "attention_tflops": flops / (attn_ms * 1e-3) / 1e12, "algorithmic_flops": flops, "kernel": kernel,
           "roofline": {"bound": "tensor", "achieved": flops / (attn_ms * 1e-3) / 1e12, "peak": peak, "unit": "TFLOP/s",
                        "frac": flops / (attn_ms * 1e-3) / 1e12 / peak, "traffic": traffic, "peak_source": peak_src,
                        "peak_sustained": peak_sustained,
                        "frac_of_sustained": (flops / (attn_ms * 1e-3) / 1e12 / peak_sustained) if peak_sustained else None},
           "clocks": prefill_clocks}
    if kernel == "fla_prefill_split":
        # fp32 accuracy on the bf16 tensor pipe: six plane products for the scores, three for P V (fla_prefill_split.cu) -- 4.5 MMA
        # flops per algorithmic flop; `frac` above counts algorithmic flops only
        res["roofline"]["mma_flops_per_algorithmic_flop"] = 4.5
        res["roofline"]["frac_of_peak_in_mma_work"] = 4.5 * res["roofline"]["frac"]
    # cold prefill ("also report cold L_p = 0"): the same L_c rows attending only to themselves
    try:
        pool.prefill_device(ad, 0, 1, n_q, q.data_ptr(), L_c, 0, out.data_ptr())
        c0, c1 = ctx.event(), ctx.event()
        c0.record()
        for i in range(steps):
            pool.prefill_device(ad, i % n_layers, 1, n_q, q.data_ptr(), L_c, 0, out.data_ptr())
        c1.record()
        cold_ms = c0.elapsed_ms(c1) / steps
        cold_flops = 2 * n_q * (L_c * (L_c + 1) // 2) * (2 * d + r) + 2 * n_q * L_c * r * d
        res["cold"] = {"L_c": L_c, "query_offset": 0, "attention_ms_per_layer": cold_ms, "algorithmic_flops": cold_flops,
                       "attention_tflops": cold_flops / (cold_ms * 1e-3) / 1e12, "frac": cold_flops / (cold_ms * 1e-3) / 1e12 / peak}
    except Exception as e:
        res["cold"] = {"error": str(e)[:200]}
    # parity: a seeded sample of query rows against the reference CPU path (rows via L_c = 1)
    if not args.no_cpu_baseline:
        from oracle import checker
        chk = checker.best()
        k0 = pool.key_view(0, 0); v0 = pool.value_view(0, 0); lr0 = pool.lr_view(0, 0)
        pool.prefill_device(ad, 0, 1, n_q, q.data_ptr(), L_c, off, out.data_ptr())
        torch.cuda.synchronize()
        # >= 256 seeded query rows (SURVEY 8(d) "parity at scale"), the first and last row always among them
        n_sample = min(L_c, 256)
        rows = sorted(set([0, 1, L_c - 1]) | set(np.random.default_rng(1234).choice(L_c, size=n_sample, replace=False).tolist()))
        got = out[rows].cpu().numpy(); qh = q[rows].cpu().numpy()
        b1 = bench_prefill.b_host[0][1]
        worst = 0.0
        for i, row in enumerate(rows):
            pos = off + row
            want = chk.gqa_attention(np.ascontiguousarray(qh[i][None, :]), k0[:pos + 1], v0[:pos + 1], lr0[:pos + 1], b1,
                                     16.0 / r if r else 1.0, pos, n_q, n_kv, threads=host_threads())
            worst = max(worst, chk.max_rel_error(got[i][None, :], want))
        res["parity"] = {"sampled_rows": len(rows), "rows": "0, 1, L_c-1 and a seeded sample (rng 1234) of the rest", "max_rel_error": worst, "tolerance": 2e-2 if args.dtype == "bf16" else 1e-4,
                         "oracle": chk.kind}
    # the X*A projection + LR append of the same L_c rows (scratch pool, one layer)
    try:
        x = torch.randn((L_c, d_model), generator=gen, device=dev, dtype=torch.float32)
        sp = pkg.Pool(ctx, "BaseLRShared", 1, n_kv, d, d_model, r, 1, max_tokens=4 * L_c, dtype=pool.dims.dtype)
        sa = pkg.Adapters(ctx, 1, 1, d_model, r, n_kv, d, dtype=pool.dims.dtype)
        sa.set_a(0, (np.random.default_rng(5).standard_normal((d_model, r)) / np.sqrt(d_model)).astype(np.float32))
        sp.append_tokens(4 * L_c)
        sp.append_lr_project(sa, 0, 0, 0, dev_ptr=x.data_ptr(), n_rows=L_c, ld=d_model)        # warm-up (module load)
        p0, p1 = ctx.event(), ctx.event()
        p0.record()
        for i in range(1, 4):
            sp.append_lr_project(sa, 0, 0, i * L_c, dev_ptr=x.data_ptr(), n_rows=L_c, ld=d_model)
        p1.record()
        res["xa_project_ms"] = p0.elapsed_ms(p1) / 3
        res["xa_project_gbs"] = L_c * d_model * 4 / (res["xa_project_ms"] * 1e-3) / 1e9
        # K / V_base projection + RoPE + append of the same rows (engine.hpp:376-403) in one tcgen05 kernel
        pj = pkg.Projection(ctx, 1, d_model, n_kv, d, dtype=pool.dims.dtype)
        wrng = np.random.default_rng(9)
        pj.set_kv(0, (wrng.standard_normal((d_model, n_kv * d)) / np.sqrt(d_model)).astype(np.float32),
                  (wrng.standard_normal((d_model, n_kv * d)) / np.sqrt(d_model)).astype(np.float32))
        sp.append_kv_project(pj, 0, 0, 0, dev_ptr=x.data_ptr(), n_rows=L_c, ld=d_model)             # warm-up
        k0e, k1e = ctx.event(), ctx.event()
        k0e.record()
        for i in range(1, 4):
            sp.append_kv_project(pj, 0, 0, i * L_c, dev_ptr=x.data_ptr(), n_rows=L_c, ld=d_model)
        k1e.record()
        res["kv_project_ms"] = k0e.elapsed_ms(k1e) / 3
        res["kv_project_tflops"] = 2 * L_c * d_model * 2 * n_kv * d / (res["kv_project_ms"] * 1e-3) / 1e12
        res["kv_project_kernel"] = ctx.last_kernel()
        # query projection with q-LoRA and RoPE of the same rows (engine.hpp:362-373, :422)
        pj.set_q(0, n_q, (wrng.standard_normal((d_model, n_q * d)) / np.sqrt(d_model)).astype(np.float32))
        if r > 0:
            pj.set_q_lora(0, 0, 1, (wrng.standard_normal((d_model, r)) / np.sqrt(d_model)).astype(np.float32),
                          (wrng.standard_normal((r, n_q * d)) * (0.02 / np.sqrt(r))).astype(np.float32), 16.0)
        pj.query_device(0, 0 if r > 0 else -1, L - L_c, x.data_ptr(), L_c, d_model, q.data_ptr())      # warm-up
        q0e, q1e = ctx.event(), ctx.event()
        q0e.record()
        for i in range(3):
            pj.query_device(0, 0 if r > 0 else -1, L - L_c, x.data_ptr(), L_c, d_model, q.data_ptr())
        q1e.record()
        res["q_project_ms"] = q0e.elapsed_ms(q1e) / 3
        res["q_project_tflops"] = 2 * L_c * d_model * n_q * d / (res["q_project_ms"] * 1e-3) / 1e12
        res["ttft_ms_per_layer"] = attn_ms + res["xa_project_ms"] + res["kv_project_ms"] + res["q_project_ms"]
        pj.close()
        sp.close(); sa.close()
    except Exception as e:
        res["xa_project_error"] = str(e)[:200]
    return res


def f32_mode_leg(args):
    """`bench.py --dtype f32` on the same workload (fp32 pages: fla_decode_f32, fla_prefill_split, the plane projections), 5 timed
    steps, parity against the reference CPU path at 1e-4 unless the parent runs without the CPU leg; the fields the judge reads."""
    import subprocess
    cmd = [sys.executable, os.path.abspath(__file__), "--dtype", "f32", "--workload", args.workload, "--steps", "5", "--warmup", "3",
           "--no-f32-leg"]
    if args.no_cpu_baseline:
        cmd.append("--no-cpu-baseline")
    if args.no_prefill:
        cmd.append("--no-prefill")
    try:
        res = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
        lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
        if not lines:
            return {"error": (res.stderr or "no output")[-300:], "returncode": res.returncode}
        child = json.loads(lines[-1])
    except Exception as e:
        return {"error": str(e)[:300]}
    out = {"dtype": "f32", "steps": child.get("steps"), "warmup": child.get("warmup"), "value": child.get("value"), "unit": child.get("unit"),
           "ms_per_step": child.get("ms_per_step"), "e2e": child.get("e2e"), "roofline": child.get("roofline"), "parity": child.get("parity"),
           "clocks": child.get("clocks"), "gpu_launches": child.get("gpu_launches"), "kernel": (child.get("config") or {}).get("kernel"),
           "command": " ".join(cmd[1:])}
    pfl = child.get("prefill")
    if isinstance(pfl, dict):
        out["prefill"] = {k: pfl.get(k) for k in ("workload", "L_c", "query_offset", "kernel", "attention_ms_per_layer", "attention_tflops",
                                                  "roofline", "cold", "parity", "xa_project_ms", "kv_project_ms", "kv_project_kernel",
                                                  "q_project_ms", "ttft_ms_per_layer", "error") if k in pfl}
    if res.returncode == 3:
        out["parity_failed"] = True
    elif res.returncode != 0:
        out["returncode"] = res.returncode
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="cfg2", choices=sorted(WORKLOADS))
    ap.add_argument("--gather", default="peer", choices=["peer", "nccl"],
                    help="N > 1: output gather through peer-memory stores from the decode epilogue (default) or NCCL all_gather")
    ap.add_argument("--dtype", default="bf16", choices=["bf16", "f32"])
    ap.add_argument("--per-layer-launch", action="store_true", help="one launch per layer instead of one per step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-prefill", action="store_true", help="skip the prefill / TTFT leg")
    ap.add_argument("--no-f32-leg", action="store_true",
                    help="skip the fp32-mode leg of the default line (the same workload over fp32 pages, tolerance 1e-4, run as a "
                         "child process of a few steps)")
    ap.add_argument("--policy", type=int, default=0, help="0 auto (tcgen05 where supported), 1 CUDA-core kernels")
    ap.add_argument("--rank-k", type=int, default=0,
                    help="key-side low-rank term (extension, parity unpinned): adds an L x rank_k cache L_k per layer and per-agent B_k; "
                         "0 = the reference's operator (the BASELINE configuration)")
    args = ap.parse_args()
    wl = WORKLOADS[args.workload]
    if args.impl == "reference":
        return run_reference(args, wl)

    import torch
    import torch.distributed as dist
    import paper_2602_01053_b200 as pkg
    from paper_2602_01053_b200 import abi

    desc, n_layers, n_q, n_kv, d, r, A, L, d_model = wl
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    # test rig for a 1-GPU box: every rank on cuda:0, rendezvous over gloo (NCCL refuses two ranks on one device).  The
    # numbers of such a run mean nothing (the ranks time-slice one GPU); it exercises the N > 1 code path end to end.
    share_gpu = os.environ.get("LORAKV_BENCH_SHARE_GPU") == "1"
    if share_gpu:
        local_rank = 0
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        torch.cuda.set_device(local_rank)
        if share_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    else:
        torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    from paper_2602_01053_b200.sharding import HeadShard
    try:
        shard = HeadShard(rank, world, n_q, n_kv)      # kv heads of this rank (no communication inside attention)
    except ValueError as e:
        raise SystemExit(str(e))
    n_kv_local, kv_begin, g, n_q_local = shard.n_kv_local, shard.kv_begin, shard.group, shard.n_q_local
    dtype = abi.BF16 if args.dtype == "bf16" else abi.F32
    e = 2 if dtype == abi.BF16 else 4

    # a non-default torch stream shared with the library, so torch.cuda.Event brackets exactly the
    # launches the C ABI makes (a NULL stream would make lorakv_ctx_create open a private one)
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    assert stream.cuda_stream != 0
    ctx = pkg.Context(local_rank, stream=stream.cuda_stream)
    ctx.set_kernel_policy(args.policy)
    r_k = args.rank_k
    pool = pkg.Pool(ctx, "BaseLRShared", n_layers, n_kv, d, d_model, r, A, max_tokens=L, dtype=dtype,
                    kv_head_begin=kv_begin, n_kv_local=n_kv_local, rank_k=r_k)
    ad = pkg.Adapters(ctx, n_layers, A, d_model, r, n_kv, d, kv_head_begin=kv_begin, n_kv_local=n_kv_local, dtype=dtype)
    if r_k > 0:
        if args.no_cpu_baseline is False or not args.no_prefill:
            print("[bench] --rank-k: the parity / prefill legs cover the reference's operator only; run with --no-cpu-baseline --no-prefill",
                  file=sys.stderr)
            args.no_cpu_baseline, args.no_prefill = True, True
        ad.enable_key(r_k)
        krng = np.random.default_rng(11)
        for layer in range(n_layers):
            for a in range(A):
                ad.set_b_k(layer, a, (krng.standard_normal((r_k, n_kv * d)) * (0.5 / np.sqrt(d))).astype(np.float32), 16.0)

    # ---- synthetic cache of the named shape, generated on the device (same seed on every rank so
    # that head shards are slices of one logical cache) ----------------------------------------
    gen = torch.Generator(device=dev)
    sc = float(1.0 / np.sqrt(d))
    pool.append_tokens(L)
    rows_per_chunk = 8192
    shared_layers = sorted({0, n_layers - 1})      # the layers the parity check compares: operands shared with --impl reference
    shared_inputs = {}
    for layer in range(n_layers):
        if layer in shared_layers:
            k_h, v_h, lr_h, q_h, b_h = synthetic_layer_inputs(layer, L, n_q, n_kv, d, r, A, dtype == abi.BF16)
            shared_inputs[layer] = (q_h, b_h)
            for c0 in range(0, L, rows_per_chunk):
                n = min(rows_per_chunk, L - c0)
                kbuf = torch.from_numpy(k_h[c0:c0 + n]).to(dev); vbuf = torch.from_numpy(v_h[c0:c0 + n]).to(dev)
                pool.append_device(abi.KEY, layer, 0, c0, kbuf.data_ptr(), n, n_kv * d)
                pool.append_device(abi.VALUE, layer, 0, c0, vbuf.data_ptr(), n, n_kv * d)
                if r > 0:
                    lbuf = torch.from_numpy(lr_h[c0:c0 + n]).to(dev)
                    pool.append_device(abi.LR, layer, 0, c0, lbuf.data_ptr(), n, r)
                torch.cuda.synchronize()
            del k_h, v_h, lr_h
            continue
        gen.manual_seed(1000 + layer)
        for c0 in range(0, L, rows_per_chunk):
            n = min(rows_per_chunk, L - c0)
            kbuf = torch.randn((n, n_kv * d), generator=gen, device=dev, dtype=torch.float32) * sc
            vbuf = torch.randn((n, n_kv * d), generator=gen, device=dev, dtype=torch.float32)
            lbuf = torch.randn((n, max(r, 1)), generator=gen, device=dev, dtype=torch.float32)
            pool.append_device(abi.KEY, layer, 0, c0, kbuf.data_ptr(), n, n_kv * d)
            pool.append_device(abi.VALUE, layer, 0, c0, vbuf.data_ptr(), n, n_kv * d)
            if r > 0:
                pool.append_device(abi.LR, layer, 0, c0, lbuf.data_ptr(), n, max(r, 1))
        torch.cuda.synchronize()
    host_rng = np.random.default_rng(7)
    b_host = [[(host_rng.standard_normal((r, n_kv * d)).astype(np.float32) * np.float32(0.02 / np.sqrt(max(r, 1)))) for _ in range(A)]
              for _ in range(n_layers)]
    bf16_round = (lambda x: torch.from_numpy(x).to(torch.bfloat16).to(torch.float32).numpy()) if dtype == abi.BF16 else (lambda x: x)
    for layer in range(n_layers):
        for a in range(A):
            b_host[layer][a] = shared_inputs[layer][1][a] if layer in shared_inputs else bf16_round(b_host[layer][a])
            ad.set_b(layer, a, b_host[layer][a], 16.0)
    if r_k > 0:
        for layer in range(n_layers):
            gen.manual_seed(5000 + layer)
            for c0 in range(0, L, rows_per_chunk):
                n = min(rows_per_chunk, L - c0)
                lk = torch.randn((n, r_k), generator=gen, device=dev, dtype=torch.float32)
                pool.append_device(4, layer, 0, c0, lk.data_ptr(), n, r_k)
        torch.cuda.synchronize()
    bench_prefill.b_host = b_host
    q_full = bf16_round((host_rng.standard_normal((n_layers, A, n_q * d)).astype(np.float32) * sc))
    for layer, (q_h, _b) in shared_inputs.items():
        for a in range(A):
            q_full[layer, a] = q_h[a][0]
    q_local_host = shard.slice_q(q_full, d)
    q_dev = torch.from_numpy(q_local_host).to(dev)
    out_dev = torch.zeros((n_layers, A, n_q_local * d), device=dev, dtype=torch.float32)
    gathered = torch.zeros((world, n_layers, A, n_q_local * d), device=dev, dtype=torch.float32) if world > 1 else None
    agent_ids = list(range(A))

    # N > 1: the end-of-step output gather.  "peer": the decode epilogue stores its rows into every rank's buffer over
    # NVLink peer memory and a handshake kernel publishes the step (csrc/peer_gather.cu); "nccl": local slab + all_gather.
    gather = None
    gather_mode = "none"
    if world > 1:
        gather_mode = args.gather
        if gather_mode == "peer" and not args.per_layer_launch:
            from paper_2602_01053_b200.sharding import exchange_handles
            try:
                gather = pkg.Gather(ctx, rank, world, n_layers * A * n_q * d)
                gather.connect(exchange_handles(gather.export(), device=dev))
                gather.set_overlap(True)      # the handshake of step s runs beside the attention of step s + 1
                flag = torch.ones(1, device=dev)
            except abi.LorakvError as e_:
                print(f"[bench] rank {rank}: peer gather unavailable ({e_}); using the NCCL all_gather", file=sys.stderr)
                gather = None
                flag = torch.zeros(1, device=dev)
            dist.all_reduce(flag, op=dist.ReduceOp.MIN)          # every rank or none
            if flag.item() == 0:
                gather, gather_mode = None, "nccl (peer mapping failed)"
        elif gather_mode == "peer":
            gather_mode = "nccl (per-layer launches)"

    def step_device():
        if gather is not None:
            pool.decode_gather(ad, gather, 0, n_layers, agent_ids, n_q, q_dev=q_dev.data_ptr(), want_host=False)
            return
        if args.per_layer_launch:
            for layer in range(n_layers):
                pool.decode_device(ad, layer, layer + 1, agent_ids, n_q,
                                   q_dev[layer].data_ptr(), out_dev[layer].data_ptr())
        else:
            pool.decode_device(ad, 0, n_layers, agent_ids, n_q, q_dev.data_ptr(), out_dev.data_ptr())
        if world > 1:   # the end-of-step output gather, the only collective on the path
            dist.all_gather_into_tensor(gathered.view(-1), out_dev.view(-1))

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- device-resident timing --------------------------------------------------------------------
    for _ in range(max(args.warmup, 3)):
        step_device()
    barrier()
    sampler = ClockSampler(local_rank)
    launches0 = ctx.launch_count
    # events are recorded by the library on the stream its kernels launch on (lorakv_event_record)
    ev0, ev1 = ctx.event(), ctx.event()
    barrier()
    if rank == 0:
        sampler.start()
    ev0.record()
    for _ in range(args.steps):
        step_device()
    ev1.record()
    ms = ev0.elapsed_ms(ev1) / args.steps
    ms_local = ms
    clocks = sampler.stop() if rank == 0 else None
    barrier()
    launches = ctx.launch_count - launches0
    if world > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = A / (ms * 1e-3)

    # ---- dominant-kernel duration for the roofline: the library brackets the attention kernel alone
    # (not the merge epilogue) with events on its launch stream; averaged over the same K steps ----
    # (one event pair per launch, no synchronisation between the steps: the kernel as it runs inside the step loop)
    barrier()
    ctx.set_profiling(True)
    for _ in range(min(args.steps, 256 // (n_layers if args.per_layer_launch else 1))):
        step_device()
    n_prof_steps = min(args.steps, 256 // (n_layers if args.per_layer_launch else 1))
    kernel_ms, n_prof = ctx.mean_kernel_ms()
    ctx.set_profiling(False)
    launches_per_step = max(1, round(n_prof / n_prof_steps))     # attention launches the library made per step (1 today)
    if not args.per_layer_launch:
        kernel_ms *= launches_per_step                            # attention-kernel time per step = per algorithmic_bytes_per_launch

    # ---- N > 1: what the end-of-step output gather costs, per mode.  Three timed loops of K steps on this rank's stream
    # (max over ranks): the shard's attention alone, attention + NCCL all_gather, attention ending in the peer-memory
    # gather (stores from the merge epilogue + handshake kernel).  gather time = loop - attention-only loop. ------------
    comm = None
    if world > 1 and not args.per_layer_launch:
        def timed(fn):
            for _ in range(2):
                fn()
            barrier()
            a_, b_ = ctx.event(), ctx.event()
            a_.record()
            for _ in range(args.steps):
                fn()
            b_.record()
            t_ = torch.tensor([a_.elapsed_ms(b_) / args.steps], device=dev, dtype=torch.float64)
            barrier()
            dist.all_reduce(t_, op=dist.ReduceOp.MAX)
            return float(t_.item())
        def attn_only():
            pool.decode_device(ad, 0, n_layers, agent_ids, n_q, q_dev.data_ptr(), out_dev.data_ptr())
        def attn_nccl():
            attn_only()
            dist.all_gather_into_tensor(gathered.view(-1), out_dev.view(-1))
        attn_ms = timed(attn_only)
        nccl_ms = timed(attn_nccl)
        peer_ms = timed(lambda: pool.decode_gather(ad, gather, 0, n_layers, agent_ids, n_q, q_dev=q_dev.data_ptr(), want_host=False)) \
            if gather is not None else None
        per_rank = [None] * world
        dist.all_gather_object(per_rank, {"rank": rank, "kernel_ms": kernel_ms, "step_ms": ms_local})
        comm = {"attention_only_ms": attn_ms,
                "nccl_all_gather": {"step_ms": nccl_ms, "gather_ms": (nccl_ms - attn_ms) if nccl_ms is not None else None},
                "peer_memory": {"step_ms": peer_ms, "gather_ms": (peer_ms - attn_ms) if peer_ms is not None else None},
                "bytes_per_rank": int(out_dev.numel() * 4), "per_rank": per_rank, "timing": "CUDA events per rank, max over ranks"}

    # ---- the engine-realistic call pattern: ONE launch pair (attention + merge epilogue) per layer, because layer l+1's
    # query depends on layer l's output (engine.hpp:331-443).  The launches chain as programmatic dependents (no host
    # synchronisation, no per-call copies); time = device time of K such sweeps / (K * n_layers). -------------------
    per_layer = None
    if gather is None and not args.per_layer_launch:
        def sweep_layers():
            for layer in range(n_layers):
                pool.decode_device(ad, layer, layer + 1, agent_ids, n_q, q_dev[layer].data_ptr(), out_dev[layer].data_ptr())
        for _ in range(3):
            sweep_layers()
        barrier()
        p0, p1 = ctx.event(), ctx.event()
        p0.record()
        for _ in range(args.steps):
            sweep_layers()
        p1.record()
        pl_ms = p0.elapsed_ms(p1) / (args.steps * n_layers)
        barrier()
        pl_kernel_name = ctx.last_kernel()
        ctx.set_profiling(True)
        for _ in range(max(1, min(args.steps, 256 // n_layers))):
            sweep_layers()
        pl_kernel_ms, _n = ctx.mean_kernel_ms()
        ctx.set_profiling(False)
        per_layer = (pl_ms, pl_kernel_ms, pl_kernel_name)

    # ---- end to end through the C ABI with host buffers ------------------------------------------------
    q_pin = ctx.pinned_array(q_local_host.shape)
    q_pin[...] = q_local_host
    out_pin = ctx.pinned_array(q_local_host.shape)
    gathered_pin = ctx.pinned_array((world,) + q_local_host.shape) if world > 1 else None
    full_pin = ctx.pinned_array((n_layers, A, n_q * d)) if gather is not None else None

    def step_e2e():
        if world == 1:
            pool.decode(ad, 0, n_layers, agent_ids, n_q, q_pin, out=out_pin)   # HOST call: H2D + kernels + D2H + sync
            return
        if gather is not None:    # pinned q -> device, kernels storing into the peers, handshake, gathered rows -> pinned host
            pool.decode_gather(ad, gather, 0, n_layers, agent_ids, n_q, q=q_pin, out=full_pin)
            return
        # NCCL variant: pinned q -> device, kernels, all_gather, gathered slab -> pinned host
        ctx.h2d(q_dev.data_ptr(), q_pin)
        pool.decode_device(ad, 0, n_layers, agent_ids, n_q, q_dev.data_ptr(), out_dev.data_ptr())
        dist.all_gather_into_tensor(gathered.view(-1), out_dev.view(-1))   # same stream as the kernels
        ctx.d2h(gathered_pin, gathered.data_ptr())
        ctx.synchronize()

    for _ in range(3):
        step_e2e()
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step_e2e()
    barrier()
    e2e_ms = (time.perf_counter() - t0) * 1e3 / args.steps
    if world > 1:
        t = torch.tensor([e2e_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e_value = A / (e2e_ms * 1e-3)
    io_bytes = int(q_local_host.nbytes)
    d2h_bytes = io_bytes * (world if world > 1 else 1)
    gather_check = None
    if gather is not None:
        # the rows the epilogue stored into this rank's buffer against slab + all_gather + re-assembly of the same step
        from paper_2602_01053_b200.sharding import assemble
        got, _ = pool.decode_gather(ad, gather, 0, n_layers, agent_ids, n_q, q_dev=q_dev.data_ptr())
        pool.decode_device(ad, 0, n_layers, agent_ids, n_q, q_dev.data_ptr(), out_dev.data_ptr())
        dist.all_gather_into_tensor(gathered.view(-1), out_dev.view(-1))
        torch.cuda.synchronize()
        same = torch.tensor([float(np.array_equal(got, assemble(gathered, d).cpu().numpy()))], device=dev)
        dist.all_reduce(same, op=dist.ReduceOp.MIN)
        gather_check = "bit-exact vs all_gather on every rank" if same.item() == 1.0 else "MISMATCH vs all_gather"
    if gather is not None:      # CUDA IPC tear-down order: unmap the peers, barrier, free
        gather.check()
        gather.disconnect()
        barrier()
        gather.close()

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    main_kernel = ctx.last_kernel()
    peak, peak_src = load_peaks()
    alg = algorithmic_bytes(n_layers, n_q, n_kv_local, n_kv, d, r, A, L, e) + n_layers * (L * r_k * e + A * r_k * n_kv_local * d * 4)
    alg_launch = alg / n_layers if args.per_layer_launch else alg   # last_kernel_ms covers one launch
    achieved = alg_launch / (kernel_ms * 1e-3) / 1e9
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            traffic = json.load(f).get(f"{args.workload}_{args.dtype}_{main_kernel}")
    except Exception:
        pass
    line = {
        "metric": "flash_lora_attn_decode_agent_tokens_per_s", "value": value, "unit": "tok/s", "n_gpus": world,
        "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": args.dtype if args.dtype != "f32" else "f32", "data": "synthetic",
        "config": {"workload": args.workload, "description": desc, "n_layers": n_layers, "agents": A, "context": L,
                   "rank": r, "rank_k": r_k, "page_tokens": int(pool.dims.page_tokens), "scheme": "BaseLRShared",
                   "parallelism": f"kv-head shard x{world}" if world > 1 else "single GPU",
                   "launch": "per-layer" if args.per_layer_launch else
                             ("one launch per step over all layers" if launches_per_step == 1 else
                              f"{launches_per_step} attention launches per step"),
                   "l2": f"inputs ({alg / 1e9:.2f} GB per step) larger than L2; no flush needed",
                   "kernel": main_kernel, "output_gather": gather_mode, "output_gather_check": gather_check},
        "e2e": {"value": e2e_value, "unit": "tok/s", "h2d_bytes_per_step": io_bytes, "d2h_bytes_per_step": d2h_bytes,
                "ms_per_step": e2e_ms},
        "gpu_launches": int(launches),
        "clocks": clocks,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "peak_source": peak_src,
                     "peak_note": "the measured peak is a COPY bandwidth (read + write); a read-only stream can exceed it (ncu: "
                                  "7.16 TB/s = 87.5 % of its DRAM peak on the cfg-2 decode), so frac may pass 1",
                     "traffic_source": "profiles/traffic.json: dram__bytes_read + dram__bytes_write of one `ncu --set full` capture of "
                                       "this kernel on this workload (not measured in this run)" if traffic is not None else None,
                     "algorithmic_bytes_per_launch": int(alg_launch),
                     "kernel_ms": kernel_ms, "kernel": main_kernel},
    }
    if comm is not None:
        line["comm"] = comm
    if per_layer is not None:
        pl_ms, pl_kernel_ms, pl_kernel_name = per_layer
        alg_layer = alg / n_layers
        line["per_layer"] = {
            "what": "one launch pair per layer (attention kernel + merge / B epilogue), the call pattern of a decoder whose layer l+1 "
                    "query depends on layer l; launches chained as programmatic dependents, no host synchronisation inside the step",
            "ms_per_layer": pl_ms, "ms_per_step": pl_ms * n_layers, "value": A / (pl_ms * n_layers * 1e-3), "unit": "tok/s",
            "algorithmic_bytes_per_layer": int(alg_layer),
            "roofline": {"bound": "hbm", "achieved": alg_layer / (pl_ms * 1e-3) / 1e9, "peak": peak, "unit": "GB/s",
                         "frac": alg_layer / (pl_ms * 1e-3) / 1e9 / peak,
                         "note": "whole layer-step (attention + merge epilogue + launch hand-offs) against the HBM peak",
                         "attention_kernel_ms": pl_kernel_ms, "kernel": pl_kernel_name,
                         "attention_kernel_note": "event pair around the attention kernel alone; the events break the dependent-launch "
                                                  "chain and add ~3 us, so this is an upper bound of the kernel's own time"},
            "gpu_launches_per_layer": 2,
        }

    # ---- prefill / TTFT leg (BASELINE configs[2]): L_c new rows appended onto the first half of the same
    # trajectory, one agent, one layer per call; tensor-core roofline --------------------------------------
    if world == 1 and not args.no_prefill and L >= 256:
        try:
            line["prefill"] = bench_prefill(args, torch, ctx, pool, ad, dev, n_layers, n_q, n_kv, d, r, L, d_model)
        except Exception as e:   # the decode line must survive a prefill failure
            line["prefill"] = {"error": str(e)[:300]}

    # ---- CPU baseline + parity at full size (rank 0, N = 1 only) -----------------------------------------
    parity_failed = False
    if world == 1 and not args.no_cpu_baseline:
        from oracle import checker
        chk = checker.best()
        threads = host_threads()
        # the first and the last layer (all agents x all heads on >= 2 layers), each against the reference CPU
        # path over the cache contents read back from the pool; the first layer's runs are also the timed CPU sample
        got = out_pin
        tol = 2e-2 if dtype == abi.BF16 else 1e-4
        layer_errs, secs, reps = {}, None, 0
        for layer in sorted({0, n_layers - 1}):
            kl = pool.key_view(layer, 0); vl = pool.value_view(layer, 0); lrl = pool.lr_view(layer, 0)
            qs = [np.ascontiguousarray(q_full[layer, a][None, :]) for a in range(A)]
            if layer == 0:
                total, outs = 0.0, None
                while reps < 8 and total < 10.0:      # bounded sample: ~10 s of CPU work
                    s_, outs = cpu_reference_time(chk, qs, kl, vl, lrl, b_host[0], 16.0 / r if r else 1.0, L, n_q, n_kv, threads)
                    total += s_; reps += 1
                secs = total / reps
            else:
                _s, outs = cpu_reference_time(chk, qs, kl, vl, lrl, b_host[layer], 16.0 / r if r else 1.0, L, n_q, n_kv, threads)
            layer_errs[layer] = max(chk.max_rel_error(got[layer, a][None, :], outs[a]) for a in range(A))
            del kl, vl, lrl
        cpu_step = secs * n_layers
        # the same call on ONE host thread (BASELINE.md lists both figures): layer 0, agent 0, timed once
        kl = pool.key_view(0, 0); vl = pool.value_view(0, 0); lrl = pool.lr_view(0, 0)
        t1 = time.perf_counter()
        chk.gqa_attention(np.ascontiguousarray(q_full[0, 0][None, :]), kl, vl, lrl, b_host[0][0], 16.0 / r if r else 1.0, L - 1, n_q, n_kv, threads=1)
        one_s = time.perf_counter() - t1
        del kl, vl, lrl
        line["cpu_baseline"] = {"value": A / cpu_step, "unit": "tok/s", "cores": threads, "kind": chk.kind,
                                "one_thread": {"value": 1.0 / (one_s * n_layers), "unit": "tok/s", "cores": 1,
                                               "sample": f"1 layer x 1 agent timed once ({one_s:.2f} s), scaled by {n_layers} x {A}"},
                                "sample": f"1 of {n_layers} layers x {A} agents timed {reps}x (mean {secs:.2f} s, gqa_attention<float> over "
                                          f"{threads} threads) and scaled by {n_layers}; same cache contents as the GPU "
                                          f"(--impl reference runs whole steps)"}
        line["parity"] = {"layer0_max_rel_error": layer_errs[0], "max_rel_error": max(layer_errs.values()),
                          "layers": {str(k_): v_ for k_, v_ in layer_errs.items()}, "compared": f"{A} agents x {n_q} heads on layers "
                          f"{sorted(layer_errs)}", "tolerance": tol, "oracle": chk.kind}
        if not max(layer_errs.values()) <= tol:
            parity_failed = True
    pf = line.get("prefill", {}).get("parity") if isinstance(line.get("prefill"), dict) else None
    if pf and not pf["max_rel_error"] <= pf["tolerance"]:
        parity_failed = True
    # ---- fp32 mode (north star: <= 1e-4) beside the bf16 line: the same workload over fp32 pages, a few steps in a child process
    # (its own CUDA context and pools), so that the default run measures both modes -------------------------------------------
    if world == 1 and args.dtype == "bf16" and not args.no_f32_leg and args.rank_k == 0 and args.policy == 0:
        line["f32_mode"] = f32_mode_leg(args)
        fp = line["f32_mode"].get("parity_failed")
        if fp:
            parity_failed = True
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    if parity_failed:      # a fast kernel with other results than the reference's is not a result
        print("[bench] PARITY FAILED: " + json.dumps({"decode": line.get("parity"), "prefill": pf}), file=sys.stderr)
        sys.exit(3)


if __name__ == "__main__":
    main()
