"""Top stall-sampled SASS instructions of an ncu source-page CSV (--page source --csv --print-source sass).
python tools/sass_hot.py file.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top_n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
h = rows[1]
ai, si = h.index("Address"), h.index("Source")
wi, ei = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
ins = [(int(r[wi] or 0), int(r[ei] or 0), r[ai][-5:], r[si].strip()) for r in rows[2:] if len(r) > ei]
tot = sum(x[0] for x in ins)
print("total samples", tot, "instructions", len(ins))
for i in sorted(sorted(range(len(ins)), key=lambda i: -ins[i][0])[:top_n]):
    w, e, a, s = ins[i]
    print(f"{i:5d} {a} {w:6d} {100 * w / tot:5.1f}% exec={e:9d}  {s[:90]}")
