"""Find backward-branch loops in a cuobjdump -sass listing and histogram their bodies.

usage: python tools/sass_loops.py file.sass [min_body_instructions]
"""
import collections
import re
import sys

lines = open(sys.argv[1]).read().splitlines()
minb = int(sys.argv[2]) if len(sys.argv) > 2 else 200
ins = []
for ln in lines:
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)(.*?);", ln)
    if m:
        ins.append((int(m.group(1), 16), m.group(3), m.group(4)))
addr_idx = {a: i for i, (a, _, _) in enumerate(ins)}
for i, (a, op, rest) in enumerate(ins):
    if op.startswith("BRA"):
        t = re.search(r"0x([0-9a-f]+)", rest)
        if not t:
            continue
        tgt = int(t.group(1), 16)
        if tgt < a and tgt in addr_idx and i - addr_idx[tgt] >= minb:
            body = ins[addr_idx[tgt]: i + 1]
            h = collections.Counter(o.split(".")[0] for _, o, _ in body)
            print(f"loop 0x{tgt:x}..0x{a:x}: {len(body)} instructions")
            print("  " + ", ".join(f"{k} {v}" for k, v in h.most_common(30)))
