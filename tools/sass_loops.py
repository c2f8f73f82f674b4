"""Per-loop instruction mix of a SASS dump (tuning aid): python tools/sass_loops.py file.sass"""
import re
import sys
from collections import Counter

L = open(sys.argv[1]).read().splitlines()
addr = {}
ins = []
for l in L:
    m = re.search(r'/\*([0-9a-f]{4,5})\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_.]+)([^;]*);', l)
    if m:
        a = int(m.group(1), 16)
        ins.append((a, m.group(3), m.group(4)))
for a, op, rest in ins:
    if op.startswith("BRA"):
        t = re.search(r'0x([0-9a-f]+)', rest)
        if t and int(t.group(1), 16) < a:
            lo = int(t.group(1), 16)
            body = [o for (x, o, _) in ins if lo <= x <= a]
            n_lds = sum(1 for o in body if o == "LDS")
            if n_lds >= 8:
                c = Counter(o.split(".")[0] for o in body)
                print(f"loop {lo:#x}-{a:#x}: {len(body)} instr, LDS {n_lds}:", c.most_common(14))
