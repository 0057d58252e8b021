"""Per-phase breakdown of an `ncu --page source --csv` (SASS) export: warp-stall samples and
executed warp instructions between CTA barriers, and samples per opcode."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
blocks, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = [r[1]]
        blocks.append(cur)
    elif cur is not None:
        cur.append(r)
for b in blocks[:1]:
    hdr = b[1]
    data = [r for r in b[2:] if len(r) == len(hdr)]
    si, src, ie = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source"), hdr.index("Instructions Executed")
    tot = sum(int(r[si] or 0) for r in data)
    print(b[0][:70], "samples", tot, "warp-instr", sum(int(r[ie] or 0) for r in data))
    seg, c, ci, start, ops = [], 0, 0, 0, {}
    for n, r in enumerate(data):
        s = int(r[si] or 0)
        c += s
        ci += int(r[ie] or 0)
        t = r[src].split()
        op = (t[1] if t and t[0].startswith("@") else (t[0] if t else "")).split(".")[0]
        ops[op] = ops.get(op, 0) + s
        if "BAR" in r[src] or n == len(data) - 1:
            seg.append((start, n, c, ci))
            c = ci = 0
            start = n + 1
    for a, e, c, i in seg:
        if c > tot * 0.01:
            print(f"  sass {a}-{e}: {c / tot * 100:.1f}% samples, {i / 1e6:.1f}M warp-instr")
    print(" ", sorted(ops.items(), key=lambda kv: -kv[1])[:16])
