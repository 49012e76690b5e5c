"""Condensed SASS listing of one kernel: `python tools/sass_ops.py file.sass [start_hex end_hex]`.
Prints opcode counts of the range and the positions of long-latency ops (SHFL, LDS, STG, BAR)."""
import re, sys
from collections import Counter
lines = open(sys.argv[1]).read().splitlines()
ins = []
for l in lines:
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
    if not m:
        continue
    addr = int(m.group(1), 16)
    body = m.group(2).strip()
    body = re.sub(r"^@!?U?P\w+\s+", "", body)
    op = body.split()[0]
    ins.append((addr, op, body))
lo = int(sys.argv[2], 16) if len(sys.argv) > 2 else 0
hi = int(sys.argv[3], 16) if len(sys.argv) > 3 else 1 << 40
sel = [x for x in ins if lo <= x[0] < hi]
c = Counter(op for _, op, _ in sel)
print(len(sel), "instructions")
print(", ".join(f"{k} {v}" for k, v in c.most_common(45)))
marks = []
for i, (a, op, b) in enumerate(sel):
    if op.startswith(("SHFL", "LDS", "STG", "BAR", "ATOMS", "RED", "LDG", "STS", "BRA")):
        marks.append(f"{i}:{op}")
print(" ".join(marks))
