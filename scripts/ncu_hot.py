"""Hottest SASS lines of an ncu source-page CSV (dev tool).
  ncu -i rep --page source --csv --print-source sass > src.csv; python scripts/ncu_hot.py src.csv [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
data = rows[2:]
S = idx["Warp Stall Sampling (All Samples)"]
E = idx["Instructions Executed"]
tot = sum(float(r[S] or 0) for r in data)
toti = sum(float(r[E] or 0) for r in data)
print(f"total samples {tot:.0f}, warp instructions {toti:.3e}")
# opcode histogram of executed instructions
from collections import Counter
c = Counter()
cs = Counter()
for r in data:
    op = r[idx["Source"]].strip().split()[0] if r[idx["Source"]].strip() else "?"
    if op.startswith("@"):
        op = r[idx["Source"]].strip().split()[1]
    op = op.split(".")[0]
    c[op] += float(r[E] or 0)
    cs[op] += float(r[S] or 0)
print("executed by opcode:", ", ".join(f"{k} {v / toti:.1%}" for k, v in c.most_common(18)))
print("stall samples by opcode:", ", ".join(f"{k} {v / tot:.1%}" for k, v in cs.most_common(12)))
top = sorted(data, key=lambda r: -float(r[S] or 0))[:n]
for r in top:
    print(f"{float(r[S]) / tot:6.1%} {r[idx['Address']][-5:]} {r[idx['Source']].strip()[:70]:70s} exec {r[E]}")
