"""Per-source-line totals (instructions executed, stall samples) from an ncu
source page exported with `--page source --csv --print-source cuda,sass`.

usage: ncu -i rep --page source --csv --print-source cuda,sass > src.csv
       python tools/ncu_lines.py src.csv [top]
"""
import collections
import csv
import sys

top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
rows = list(csv.reader(open(sys.argv[1])))
cur_file, hdr = None, None
inst = collections.Counter()
samp = collections.Counter()
text = {}
last_line = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = {h: i for i, h in enumerate(r)}
        continue
    if hdr is None or len(r) < 5:
        continue
    # cuda source rows carry a line number in column 0; sass rows below them have an address
    if r[0].strip().isdigit():
        last_line = (cur_file, int(r[0]))
        text[last_line] = r[1].strip()[:90]
        try:
            inst[last_line] += float((r[hdr["Instructions Executed"]] or "0").replace(",", ""))
            samp[last_line] += float((r[hdr["Warp Stall Sampling (All Samples)"]] or "0").replace(",", ""))
        except (ValueError, KeyError, IndexError):
            pass
tot_i = sum(inst.values()) or 1
tot_s = sum(samp.values()) or 1
print(f"warp instructions {tot_i:.3e}, stall samples {tot_s:.0f}")
for key, v in inst.most_common(top):
    print(f"{v / tot_i * 100:5.1f}% inst {samp[key] / tot_s * 100:5.1f}% samp  {key[0]}:{key[1]}  {text.get(key, '')}")
