"""Stall-reason breakdown per barrier-delimited phase of an `ncu --page source --csv --print-source sass`
export: which stall dominates each phase (samples per stall_* column)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = [r for r in rows[2:] if len(r) == len(hdr)]
si, src = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source")
cols = [i for i, h in enumerate(hdr) if h.startswith("stall_")]
tot = sum(int(r[si] or 0) for r in data)
seg, acc, start = [], None, 0
for n, r in enumerate(data):
    if acc is None:
        acc = [0] * len(cols)
        c = 0
    c += int(r[si] or 0)
    for k, i in enumerate(cols):
        acc[k] += int(r[i] or 0)
    if "BAR.SYNC" in r[src] or n == len(data) - 1:
        if c > 0.01 * tot:
            top = sorted(zip(acc, [hdr[i] for i in cols]), reverse=True)[:6]
            print(f"sass {start}-{n}: {100 * c / tot:.1f}% samples;", ", ".join(f"{h[6:]} {100 * v / c:.0f}%" for v, h in top))
        acc, start = None, n + 1
