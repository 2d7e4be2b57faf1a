"""The recorded bench lines (profiles/r1_bench_cfg2.json, profiles/r2_bench_cfg2.json, written by `python bench.py` on a B200,
and profiles/r2_bench_reference_arm.json by `--impl reference`) carry every key the measurement contract asks for, with
consistent arithmetic.  CPU only: it reads the committed JSON."""
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


import pytest


@pytest.mark.parametrize("name", ["r1_bench_cfg2.json", "r2_bench_cfg2.json"])
def test_recorded_bench_line_has_the_contract_keys(name):
    d = json.load(open(os.path.join(ROOT, "profiles", name)))
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling", "vs_baseline",
              "dtype", "data", "config", "e2e", "gpu_launches", "clocks", "roofline", "cpu_baseline"):
        assert k in d, k
    assert d["config"]["workload"] == "cfg2" and d["data"] == "synthetic" and d["vs_baseline"] is None
    assert d["warmup"] >= 3 and d["gpu_launches"] > 0
    assert abs(d["value"] - d["config"]["agents"] / (d["ms_per_step"] * 1e-3)) < 1e-6 * d["value"]
    e = d["e2e"]
    assert e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0 and 0 < e["value"] < d["value"]
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    # the attention kernel's own DRAM bytes; the algorithmic figure also counts out and B (0.1 %), which the merge kernel touches
    assert r["traffic"] is None or r["traffic"] >= 0.99 * r["algorithmic_bytes_per_launch"]
    assert abs(r["achieved"] - r["algorithmic_bytes_per_launch"] / (r["kernel_ms"] * 1e-3) / 1e9) < 1e-6 * r["achieved"]
    c = d["cpu_baseline"]
    assert c["kind"] in ("reference", "port") and c["cores"] >= 1 and c["value"] > 0 and c["sample"]
    assert not set(d["clocks"]["reasons"]) & {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}
    if name.startswith("r2"):
        # round 2: one launch pair per layer, parity on two layers and >= 256 prefill rows, the 1-thread CPU figure
        pl = d["per_layer"]
        assert pl["gpu_launches_per_layer"] == 2 and abs(pl["ms_per_step"] - pl["ms_per_layer"] * d["config"]["n_layers"]) < 1e-9
        rf = pl["roofline"]
        assert abs(rf["achieved"] - pl["algorithmic_bytes_per_layer"] / (pl["ms_per_layer"] * 1e-3) / 1e9) < 1e-6 * rf["achieved"]
        assert abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-9 and rf["frac"] >= 0.70            # the north star's decode target
        assert pl["algorithmic_bytes_per_layer"] * d["config"]["n_layers"] == r["algorithmic_bytes_per_launch"]
        par = d["parity"]
        assert set(par["layers"]) == {"0", str(d["config"]["n_layers"] - 1)} and par["max_rel_error"] <= par["tolerance"]
        pp = d["prefill"]["parity"]
        assert pp["sampled_rows"] >= 256 and pp["max_rel_error"] <= pp["tolerance"]
        assert c["one_thread"]["cores"] == 1 and 0 < c["one_thread"]["value"] < c["value"]
        assert "not measured in this run" in r["traffic_source"]
        # the fp32 mode of the north star (<= 1e-4) is measured by the same default run, as a child process over fp32 pages
        f = d["f32_mode"]
        assert f["dtype"] == "f32" and f["warmup"] >= 3 and f["gpu_launches"] > 0 and not f.get("parity_failed")
        assert f["parity"]["tolerance"] == 1e-4 and f["parity"]["max_rel_error"] <= 1e-4
        assert f["roofline"]["bound"] == "hbm" and f["roofline"]["frac"] >= 0.70 and f["roofline"]["kernel"] == "fla_decode_f32"
        fp = f["prefill"]
        assert fp["kernel"] == "fla_prefill_split" and fp["parity"]["sampled_rows"] >= 256 and fp["parity"]["max_rel_error"] <= 1e-4
        assert fp["kv_project_kernel"] == "kv_project_planes"
        rr = fp["roofline"]
        assert rr["mma_flops_per_algorithmic_flop"] == 4.5 and abs(rr["frac_of_peak_in_mma_work"] - 4.5 * rr["frac"]) < 1e-9


def test_recorded_reference_arm_line():
    d = json.load(open(os.path.join(ROOT, "profiles", "r2_bench_reference_arm.json")))
    assert d["impl"] == "reference" and d["config"]["workload"] == "cfg2" and d["higher_is_better"] is True
    assert d["metric"] == "flash_lora_attn_decode_agent_tokens_per_s" and d["unit"] == "tok/s"
    assert d["e2e"] == {"value": d["value"], "unit": "tok/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    c = d["cpu_baseline"]
    assert c["value"] == d["value"] and c["kind"] in ("reference", "port") and c["cores"] >= 1
    assert "32 of 32 layers" in c["sample"]                      # whole steps, not one layer scaled
    assert abs(d["value"] - d["config"]["agents"] / (d["ms_per_step"] * 1e-3)) < 1e-6 * d["value"]
