"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: mean us per kernel."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
tag = sys.argv[2] if len(sys.argv) > 2 else ""
hdr, agg = None, defaultdict(list)
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        agg[d["Kernel Name"]].append(float(d["Metric Value"].replace(",", "")) / 1e3)
tot = {"op0": 0.0, "op1": 0.0}
for k, v in agg.items():
    m = sum(v) / len(v)
    print(f"{tag:10s} {k[:64]:64s} n={len(v):3d} mean_us={m:9.1f}")
    for op in ("0", "1"):
        if k.endswith(f", {op}>(fp::PathArgs<T1>)"):
            tot["op" + op] += m
print(f"{tag:10s} serial sum: fwd {tot['op0']:.1f} us, fused {tot['op1']:.1f} us")
