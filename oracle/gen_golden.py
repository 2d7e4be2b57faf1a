#!/usr/bin/env python
"""Generate tests/golden/*.npz from the REFERENCE itself (oracle/_ref, i.e. the unmodified
headers under /root/reference/proj/include compiled by oracle/Makefile).

TEST INFRASTRUCTURE ONLY.  Run in the dev container (where /root/reference exists):

    python oracle/gen_golden.py

The fixtures pin the known-answer cases of the reference's own tests for this path
(SURVEY.md section 8c): tests/test_attention.cpp seeds 31, 40-42(+100), 47, 53, 61, 83, 113, 127,
149, 151, 157, 977, the fuzz seeds 7001/7002/555, lr_mac_counts spot values, test_kvcache.cpp's
plan_core intervals / first-writer-wins / byte-ratio identities, and rng.hpp streams.
Inputs are regenerated from seeds by the tests (through the oracle's RNG, itself pinned here), so
the files stay small: they hold seeds, shapes and the reference's OUTPUTS.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import checker  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")


def random_case(chk, L, L_c, d, r, offset, seed, dtype):
    """tests/test_attention.cpp:32-43 random_case()."""
    g = lambda rows, cols, key: chk.gaussian(rows, cols, chk.child(seed, key), 1.0, dtype)
    return dict(q=g(L_c, d, 1), k=g(L, d, 2), v=g(L, d, 3), v_lr=g(L, r, 4), b_up=g(r, d, 5),
                scale=0.5, offset=offset)


# (name, L, L_c, d, r, offset, seed, b_r, b_c) -- shapes of the reference's own test cases
ATTENTION_CASES = [
    ("single_token", 1, 1, 8, 2, 0, 31, 4, 4),                 # test_attention.cpp:75-85
    ("scalar_loop_40", 12, 5, 6, 0, 7, 40, 4, 4),              # :87-99 (r = 0 variant)
    ("scalar_loop_140", 10, 10, 4, 3, 0, 140, 4, 4),           # :95 seed + 100
    ("scalar_loop_141", 10, 10, 4, 3, 0, 141, 3, 5),
    ("scalar_loop_142", 10, 10, 4, 3, 0, 142, 1, 1),
    ("first_row", 4, 4, 4, 2, 0, 53, 2, 2),                    # :120-128
    ("single_block", 24, 9, 16, 8, 15, 61, 64, 64),            # :130-135
    ("stats", 20, 8, 8, 2, 12, 83, 3, 5),                      # :196-215
    ("expand_first", 30, 11, 8, 4, 19, 113, 4, 8),             # :259-264
    ("rank0", 16, 6, 8, 0, 10, 127, 4, 4),                     # :266-272
    ("masked_977", 24, 6, 8, 2, 9, 977, 2, 3),                 # :144-175 (before the 1e6 edit)
]


def main():
    ref = checker.reference()
    if ref is None:
        raise SystemExit("oracle/_ref is not built and /root/reference is absent")
    os.makedirs(OUT, exist_ok=True)

    # ---- rng.hpp streams -----------------------------------------------------------------
    rng = {
        "seeds": np.array([0, 1, 42, 7001, 20250810, 2**63 + 12345], dtype=np.uint64),
    }
    rng["u64"] = np.stack([ref.u64(int(s), 8) for s in rng["seeds"]])
    rng["child_3"] = np.array([ref.child(int(s), 3) for s in rng["seeds"]], dtype=np.uint64)
    rng["mix_with_f022"] = np.array([ref.mix(int(s), 0xf022) for s in rng["seeds"]], dtype=np.uint64)
    rng["gauss_f64"] = np.stack([ref.gaussian(1, 16, int(s), 1.0, np.float64)[0] for s in rng["seeds"]])
    rng["gauss_f32_scaled"] = np.stack([ref.gaussian(1, 16, int(s), 0.125, np.float32)[0] for s in rng["seeds"]])
    np.savez(os.path.join(OUT, "rng.npz"), **rng)

    # ---- attention known-answer cases ----------------------------------------------------
    att = {}
    meta = []
    for name, L, L_c, d, r, off, seed, br, bc in ATTENTION_CASES:
        for dt, tag in ((np.float64, "f64"), (np.float32, "f32")):
            c = random_case(ref, L, L_c, d, r, off, seed, dt)
            args = (c["q"], c["k"], c["v"], c["v_lr"], c["b_up"], c["scale"], c["offset"])
            naive = ref.naive_attention(*args)
            flash, macs, (rmax, rden) = ref.flash_lora_attention(*args, br, bc, want_macs=True,
                                                                 want_stats=True)
            expand, emacs = ref.expand_first_attention(*args, br, bc, want_macs=True)
            key = f"{name}_{tag}"
            att[key + "_naive"] = naive
            att[key + "_flash"] = flash
            att[key + "_expand"] = expand
            att[key + "_rowmax"] = rmax
            att[key + "_rowdenom"] = rden
            att[key + "_macs"] = np.array(list(macs) + list(emacs), dtype=np.uint64)
        meta.append(dict(name=name, L=L, L_c=L_c, d=d, r=r, offset=off, seed=seed, b_r=br, b_c=bc))

    # GQA cases (test_attention.cpp:286-363): seeds 149 (3/3 heads) and 151 (4 q / 2 kv)
    for seed, n_q, n_kv in ((149, 3, 3), (151, 4, 2)):
        L, L_c, d_head, r = 12, 5, 4, 2
        for dt, tag in ((np.float64, "f64"), (np.float32, "f32")):
            g = lambda rows, cols, key: ref.gaussian(rows, cols, ref.child(seed, key), 1.0, dt)
            q, k, v = g(L_c, n_q * d_head, 1), g(L, n_kv * d_head, 2), g(L, n_kv * d_head, 3)
            v_lr, b_up = g(L, r, 4), g(r, n_kv * d_head, 5)
            out, macs = ref.gqa_attention(q, k, v, v_lr, b_up, 0.5, L - L_c, n_q, n_kv, 4, 4,
                                          want_macs=True)
            att[f"gqa_{seed}_{tag}"] = out
            att[f"gqa_{seed}_{tag}_macs"] = np.array(macs, dtype=np.uint64)

    # masked-positions case (test_attention.cpp:144-175): 1e6 keys/values beyond the boundary
    L, L_c, d, r, off = 24, 6, 8, 2, 9
    c = random_case(ref, L, L_c, d, r, off, 977, np.float64)
    c["k"][off + L_c:, :] = 1e6
    c["v"][off + L_c:, :] = 1e6
    for br in (2, 8):
        for bc in (3, 5, 64):
            att[f"masked_1e6_{br}_{bc}"] = ref.flash_lora_attention(
                c["q"], c["k"], c["v"], c["v_lr"], c["b_up"], 0.5, off, br, bc)
    np.savez(os.path.join(OUT, "attention.npz"), **att)

    # ---- fuzz statistics (test_attention.cpp:137-142,177-183; fuzz.hpp) -------------------
    fuzz = {
        "f64_40_7001_48": ref.kernel_fuzz(40, 7001, 48, "f64"),
        "f32_40_7002_48": ref.kernel_fuzz(40, 7002, 48, "f32"),
        "f64_12_555_32": ref.kernel_fuzz(12, 555, 32, "f64"),
    }

    # ---- lr_mac_counts (test_attention.cpp:217-232, acceptance.cpp:135) -------------------
    mac_rows = []
    for L, Lc, r, d in ((4096, 1, 8, 128), (100, 10, 16, 16), (32, 32, 1, 1), (32768, 1, 16, 128),
                        (65536, 1, 64, 128), (131072, 1, 32, 128), (32768, 16384, 16, 128)):
        mac_rows.append([L, Lc, r, d, *ref.lr_mac_counts(L, Lc, r, d)])

    # ---- plan_core (test_kvcache.cpp:58-114) -----------------------------------------------
    plans = []
    for scheme in ("NonShared", "FullShared", "BaseShared", "BaseLRShared", "SelectiveRecompute"):
        for length, seen, new in ((0, 0, 16), (1000, 0, 10), (1000, 1000, 1), (1000, 400, 0),
                                  (32768, 32768, 1), (16384, 0, 16384)):
            for first in ((0, 2) if scheme == "SelectiveRecompute" else (0,)):
                p = ref.plan_core(scheme, length, seen, new, first)
                plans.append(dict(scheme=scheme, length=length, seen=seen, new=new, first=first, plan=p))

    # ---- store bookkeeping (test_kvcache.cpp:116-164,189-277) -------------------------------
    def fill_rows(rows, cols, tag):
        return (tag + np.arange(rows * cols, dtype=np.float64)).reshape(rows, cols)

    stores = []
    for r in (4, 8, 16, 32):
        for d_out in (256, 1024):
            row = dict(r=r, d_out=d_out, L=24, n_layers=2, N=3, bytes={})
            for scheme in ("NonShared", "BaseShared", "BaseLRShared", "FullShared"):
                st = ref.store(scheme, 2, d_out, 4 * d_out, r, 3, np.float64)
                st.append_tokens(24)
                for layer in range(2):
                    kv = fill_rows(24, d_out, 1000.0 * layer)
                    agents = range(3) if scheme == "NonShared" else (0,)
                    for a in agents:
                        st.append_key(layer, a, 0, kv)
                        st.append_value(layer, a, 0, kv)
                    lr = fill_rows(24, r, 77.0 + layer)
                    if scheme == "BaseShared":
                        for a in range(3):
                            st.append_lr(layer, a, 0, lr)
                    if scheme == "BaseLRShared":
                        st.append_lr(layer, 0, 0, lr)
                for a in range(3):
                    st.mark_seen(a)
                row["bytes"][scheme] = st.bytes()
                row.setdefault("elements", {})[scheme] = st.allocated_elements()
            stores.append(row)

    # first-writer-wins trace (test_kvcache.cpp:116-140) recorded as (rows_before, row_begin, n) -> rows_after
    fww = []
    st = ref.store("BaseShared", 1, 4, 8, 2, 3, np.float64)
    st.append_tokens(6)
    seq = [(0, 0, 0, 6), (1, 0, 0, 6), (2, 0, 0, 6), (0, 1, 0, 6), (1, 1, 3, 5), (2, 1, 0, 6),
           (0, 2, 6, 2), (1, 2, 4, 4)]
    for which, agent, row_begin, n in seq:
        before = [st.key_view(0, agent).shape[0], st.value_view(0, agent).shape[0],
                  st.lr_view(0, agent).shape[0]][which]
        cols = 2 if which == 2 else 4
        st._append(which, 0, agent, row_begin, fill_rows(n, cols, 100.0 * agent + row_begin))
        after = [st.key_view(0, agent).shape[0], st.value_view(0, agent).shape[0],
                 st.lr_view(0, agent).shape[0]][which]
        fww.append(dict(which=which, agent=agent, row_begin=row_begin, n=n, before=before, after=after))
    gap_msg = None
    try:
        st.append_value(0, 0, 99, fill_rows(1, 4, 0.0))
    except checker.CheckerError as e:
        gap_msg = str(e)
    fww_final = dict(key=st.key_view(0, 1).tolist(), lr0=st.lr_view(0, 0).tolist(),
                     lr1=st.lr_view(0, 1).tolist(), gap_message=gap_msg, bytes=st.bytes())

    with open(os.path.join(OUT, "tables.json"), "w") as f:
        json.dump(dict(attention_cases=meta, fuzz=fuzz, lr_mac_counts=mac_rows, plans=plans,
                       store_bytes=stores, fww_trace=fww, fww_final=fww_final), f, indent=1)
    print("wrote", sorted(os.listdir(OUT)))


if __name__ == "__main__":
    main()
