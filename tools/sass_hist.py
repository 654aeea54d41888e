"""Instruction mix of an ncu source-page CSV (--page source --print-source sass):
executed warp-instructions and stall samples per opcode, and the hottest lines.

    python tools/sass_hist.py gpurun_out/symb_sass.csv [top]
"""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ia, isrc, iex, ismp = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed"), \
    hdr.index("Warp Stall Sampling (All Samples)")
ops, smp, lines = Counter(), Counter(), []
tot = tots = 0
for r in rows[2:]:
    if len(r) <= iex:
        continue
    try:
        n = int(r[iex]); s = int(r[ismp])
    except ValueError:
        continue
    src = r[isrc].strip()
    op = src.split()[0] if not src.startswith("@") else src.split()[1]
    op = op.split(".")[0]
    ops[op] += n; smp[op] += s; tot += n; tots += s
    lines.append((n, s, r[ia], src))
print(f"total warp-instructions {tot:.4e}, stall samples {tots}")
for op, n in ops.most_common(30):
    print(f"  {op:10s} {n:12d} {100 * n / tot:5.1f}%  samples {100 * smp[op] / max(tots, 1):5.1f}%")
top = int(sys.argv[2]) if len(sys.argv) > 2 else 0
for n, s, a, src in sorted(lines, reverse=True)[:top]:
    print(f"{n:12d} {s:6d} {a} {src}")
