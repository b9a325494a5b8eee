"""Executed-instruction histogram and stall breakdown from an ncu source-page CSV.

usage: ncu -i rep --page source --csv --print-source sass > src.csv
       python tools/ncu_sass_exec.py src.csv [top]
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 20
hdr = next(r for r in rows if r and r[0] == "Address")
ix = {h: i for i, h in enumerate(hdr)}
data = [r for r in rows if len(r) == len(hdr) and r[0].startswith("0x")]
seen = set()
uniq = []
for r in data:
    if r[0] not in seen:
        seen.add(r[0])
        uniq.append(r)


def num(r, c):
    try:
        return float((r[ix[c]] or "0").replace(",", ""))
    except ValueError:
        return 0.0


ex = collections.Counter()
for r in uniq:
    op = r[ix["Source"]].strip().split()
    if not op:
        continue
    o = op[0] if not op[0].startswith("@") else op[1]
    ex[o.split(".")[0]] += num(r, "Instructions Executed")
tot = sum(ex.values())
print(f"warp instructions executed: {tot:.0f}")
for o, v in ex.most_common(top):
    print(f"  {o:8s} {v / tot * 100:5.1f}%  {v:.0f}")
cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
st = {c: sum(num(r, c) for r in uniq) for c in cols}
S = sum(st.values()) or 1
print("stall samples:", ", ".join(f"{c[6:]} {v / S * 100:.1f}%" for c, v in sorted(st.items(), key=lambda kv: -kv[1])[:9]))
