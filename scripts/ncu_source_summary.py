"""Summarise an ncu --page source --csv (SASS) dump: stall totals and the
instructions with most stall samples / shared-memory conflicts."""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
def num(r, k):
    try:
        return float(r[ix[k]])
    except (ValueError, KeyError, IndexError):
        return 0.0
tot = Counter()
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
for r in data:
    for c in stall_cols:
        tot[c] += num(r, c)
all_s = sum(tot.values())
print("total samples", all_s)
for c, v in tot.most_common(10):
    print(f"  {c:28s} {v:8.0f} {100*v/max(all_s,1):5.1f}%")
ops = Counter()
for r in data:
    op = r[ix["Source"]].split()[0] if r[ix["Source"]].strip() else "?"
    if op.startswith("@"):
        op = r[ix["Source"]].split()[1]
    ops[op.split(".")[0]] += num(r, "Warp Stall Sampling (All Samples)")
print("samples by opcode:", ops.most_common(12))
top = sorted(data, key=lambda r: -num(r, "Warp Stall Sampling (All Samples)"))[:int(sys.argv[2]) if len(sys.argv) > 2 else 15]
for r in top:
    st = sorted(((num(r, c), c) for c in stall_cols), reverse=True)[:2]
    print(f"{r[ix['Address']]:>6} {num(r,'Warp Stall Sampling (All Samples)'):6.0f} {r[ix['Source']][:60]:60s} {st}")
conf = sorted(data, key=lambda r: -num(r, "L1 Wavefronts Shared Excessive"))[:8]
print("shared excessive wavefronts:")
for r in conf:
    if num(r, "L1 Wavefronts Shared Excessive") > 0:
        print(f"{r[ix['Address']]:>6} {r[ix['Source']][:60]:60s} excess={num(r,'L1 Wavefronts Shared Excessive'):.0f} ideal={num(r,'L1 Wavefronts Shared Ideal'):.0f}")
