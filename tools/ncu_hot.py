"""Top stall-sample SASS lines of an ncu source-page CSV (first kernel)."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = rows[1]
i_src, i_s = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
data = []
for r in rows[2:]:
    if len(r) < len(hdr) or r[0].startswith('"Kernel'):
        break
    try:
        data.append((int(r[i_s]), r[0][-5:], r[i_src].strip()))
    except ValueError:
        break
tot = sum(d[0] for d in data)
print("total samples", tot)
for s, a, src in sorted(data, reverse=True)[:n]:
    print(f"{s:7d} {100*s/tot:5.1f}%  {a}  {src[:90]}")
