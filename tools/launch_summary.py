"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv): per-kernel totals of the
library's own kernels (ipr::), in launch order segments.  python tools/launch_summary.py file.csv"""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    out = []
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        out.append((r[ki], v, r[h.index("Grid Size")]))
    return out


def main():
    ks = [k for k in load(sys.argv[1]) if "ipr::" in k[0]]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for name, v, grid in ks:
        key = name.split("(")[0].replace("void ", "")[:60]
        agg[key][0] += 1
        agg[key][1] += v
    tot = sum(v for _, v, _ in ks)
    for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{v / 1e6:9.3f} ms {100 * v / tot:5.1f}% {c:5d}  {k}")
    print(f"{tot / 1e6:9.3f} ms total, {len(ks)} launches")


if __name__ == "__main__":
    main()
