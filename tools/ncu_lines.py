"""Per-source-line instruction / stall shares of one kernel in an ncu report:
maps the report's SASS (page source) onto line info from nvdisasm -g of the
object file.  python tools/ncu_lines.py REPORT OBJ KERNEL_SUBSTR [top]"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile


def main(rep, obj, kname, top=40):
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(src)))
    h = rows[1]
    data = rows[2:]
    iS, iE, iW = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    with tempfile.TemporaryDirectory() as d:
        subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True)
        cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
        dis = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, cub)], capture_output=True, text=True).stdout
    lines = dis.split("\n")
    st = [i for i, l in enumerate(lines) if l.startswith(".text.") and kname in l][0]
    instrs, cur, curf = [], None, None
    for l in lines[st + 1:]:
        if l.startswith(".text."):
            break
        m = re.search(r'//## File "(.*)", line (\d+)', l)
        if m:
            curf, cur = os.path.basename(m.group(1)), int(m.group(2))
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
        if m:
            instrs.append((int(m.group(1), 16), (curf, cur), m.group(2)))
    base = int(data[0][0], 16)
    by = {int(r[0], 16) - base: (int(r[iE] or 0), int(r[iW] or 0)) for r in data}
    pl, ps = collections.Counter(), collections.Counter()
    ops = collections.Counter()
    for a, ln, txt in instrs:
        e, s = by.get(a, (0, 0))
        pl[ln] += e
        ps[ln] += s
        ops[txt.split()[0].split(".")[0] if not txt.startswith("@") else txt.split()[1].split(".")[0]] += e
    tot, tots = sum(pl.values()), sum(ps.values())
    print(f"warp-instructions {tot:.4e}")
    print("by opcode:", ", ".join(f"{o} {c / tot * 100:.1f}%" for o, c in ops.most_common(16)))
    srcs = {}
    for (f, ln), c in pl.most_common(top):
        if f and f not in srcs:
            p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_1305_5179_b200", "csrc", f)
            srcs[f] = open(p).read().split("\n") if os.path.exists(p) else []
        txt = srcs.get(f, [])[ln - 1].strip()[:95] if f and ln and srcs.get(f) else ""
        print(f"{f}:{ln:<5} {c / tot * 100:5.1f}%  stall {ps[(f, ln)] / tots * 100:5.1f}%  {txt}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4]) if len(sys.argv) > 4 else 40)
