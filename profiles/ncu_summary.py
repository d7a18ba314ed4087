"""Summarise an ncu source page (SASS) export: instruction mix and stall reasons.
usage: ncu -i X.ncu-rep --page source --csv --print-source sass > src.csv; python profiles/ncu_summary.py src.csv"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot_inst = 0
by_op = collections.Counter()
stall_tot = collections.Counter()
samples = 0
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    src = r[ix["Source"]].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    base = op.split(".")[0]
    n = int(float(r[ix["Instructions Executed"]] or 0))
    tot_inst += n
    by_op[base] += n
    samples += int(float(r[ix["Warp Stall Sampling (All Samples)"]] or 0))
    for s in stalls:
        stall_tot[s] += int(float(r[ix[s]] or 0))
print(f"warp instructions executed: {tot_inst:.4g}")
for op, n in by_op.most_common(30):
    print(f"  {op:10s} {n:14d} {100 * n / tot_inst:6.2f}%")
print(f"stall samples: {samples}")
for s, n in stall_tot.most_common(12):
    print(f"  {s:28s} {n:10d} {100 * n / max(samples, 1):6.2f}%")
