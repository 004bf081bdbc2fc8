"""Per-source-line warp-stall breakdown of an ncu source export (sass csv).

usage: ncu_stalls.py <src.csv> <nvdisasm --print-line-info dump> <mangled-kernel-substr> [N]
Prints the top lines by stall samples with their dominant stall reasons
(file:line resolved from the dump, so inlined helpers show their own file).
"""
import csv
import re
import sys
from collections import Counter, defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
iS = hdr.index("Warp Stall Sampling (All Samples)")
iE = hdr.index("Instructions Executed")
stall_cols = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
recs = [r for r in rows[2:] if len(r) >= len(hdr)]
base = int(recs[0][0], 16)
off2line, cur, inside = {}, None, False
for L in open(sys.argv[2]).read().split("\n"):
    if L.startswith(".text."):
        inside = sys.argv[3] in L
    if not inside:
        continue
    m = re.search(r'line (\d+)', L)
    if m and "//##" in L:
        f = re.search(r'File "([^"]+)"', L)
        cur = (f.group(1).split("/")[-1] if f else "?") + ":" + m.group(1)
    m = re.search(r'/\*([0-9a-f]{4,})\*/', L)
    if m and cur is not None:
        off2line[int(m.group(1), 16)] = cur
samp, exe, why = Counter(), Counter(), defaultdict(Counter)
tot_why = Counter()
for r in recs:
    ln = off2line.get(int(r[0], 16) - base, "?")
    samp[ln] += int(r[iS] or 0)
    exe[ln] += int(r[iE] or 0)
    for i, h in stall_cols:
        v = int(r[i] or 0)
        why[ln][h[6:]] += v
        tot_why[h[6:]] += v
tot = sum(samp.values())
print(f"total samples {tot}; by reason: " +
      ", ".join(f"{k} {100 * v / tot:.1f}%" for k, v in tot_why.most_common(8)))
N = int(sys.argv[4]) if len(sys.argv) > 4 else 30
for ln, s in samp.most_common(N):
    top = ", ".join(f"{k} {v}" for k, v in why[ln].most_common(3))
    print(f"{ln:22s} {100 * s / tot:5.1f}%  exec {exe[ln]:>11d}  [{top}]")
