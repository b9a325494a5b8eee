"""Table of per-kernel mean durations from tools/ab_ncu.sh output: python tools/ab_table.py file"""
import re
import sys

rows, libs = {}, []
for l in open(sys.argv[1]):
    m = re.match(r"(\S+)\s+void (?:fp::)?path_kernel<float, (?:\(int\))?(\d), (?:\(unsigned int\))?(\d+), "
                 r"(?:\(int\))?(\d)>.*mean_us=\s*([\d.]+)", l)
    if m:
        lib = m.group(1)
        if lib not in libs:
            libs.append(lib)
        rows.setdefault((int(m.group(4)), int(m.group(3))), {})[lib] = float(m.group(5))
print("op mask " + " ".join(f"{x:>12s}" for x in libs))
tot = {x: [0.0, 0.0, 0.0] for x in libs}
for (op, mask), d in sorted(rows.items()):
    print(f"{op:2d} {mask:4d} " + " ".join(f"{d.get(x, 0):12.1f}" for x in libs))
    for x in libs:
        tot[x][op] += d.get(x, 0)
print("sum fwd  " + " ".join(f"{tot[x][0]:12.1f}" for x in libs))
print("sum fused" + " ".join(f"{tot[x][1]:12.1f}" for x in libs))
