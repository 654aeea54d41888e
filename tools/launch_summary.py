"""Aggregate an ncu launch-list CSV (gpu__time_duration.sum) by kernel name.

    python tools/launch_summary.py gpurun_out/launches.csv [top]
"""
import collections
import csv
import sys


def main(path, top=25):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[h + 1:]:
        if len(r) <= vi:
            continue
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}.get(r[ui], 1e-6)
        k = r[ki].split("(")[0][:80]
        agg[k][0] += 1
        agg[k][1] += v * scale
    tot = sum(v[1] for v in agg.values())
    print(f"total {tot:.1f} ms over {sum(v[0] for v in agg.values())} launches")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        print(f"{v[1]:10.2f} ms {100 * v[1] / tot:5.1f}% {v[0]:6d}  {k}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
