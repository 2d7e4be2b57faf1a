"""Summarise an `ncu --page source --csv` export: top stall-sampled SASS instructions and a per-region
breakdown between marker instructions.  usage: ncu_src_summary.py file.csv [min_pct]"""
import csv, sys, re
rows = list(csv.reader(open(sys.argv[1])))
hdr, data = rows[1], rows[2:]
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.4
isrc, isamp, iex = hdr.index("Source"), hdr.index("# Samples"), hdr.index("Instructions Executed")
stall = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(int(r[isamp]) for r in data)
print("total samples", tot, "instructions", len(data))
for k, r in enumerate(data):
    s = int(r[isamp]); src = r[isrc].strip()
    if s >= tot * thr / 100 or re.search(r"UTCBAR|LDTM|STTM|BAR\.SYNC|SYNCS\.ARRIVE|TRYWAIT", src):
        st = sorted(((int(r[i]), hdr[i][6:]) for i in stall), reverse=True)[:2]
        print(k, s, f"{100*s/tot:.2f}%", r[iex], src[:80], st)
