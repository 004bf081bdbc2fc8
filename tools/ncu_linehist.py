"""Per-source-line stall samples of one kernel (ntt_ts.cu lines lo..hi).

usage: ncu_linehist.py <ncu sass csv> <nvdisasm dump> <mangled kernel substring> lo hi
"""
import csv, re, sys
from collections import Counter
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
i_s, i_src, i_ex = (hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source"),
                    hdr.index("Instructions Executed"))
stall_cols = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
recs = []
for r in rows[2:]:
    if len(r) < len(hdr): break
    try: recs.append((int(r[0], 16), int(r[i_s]), int(r[i_ex]), [int(r[i]) for i, _ in stall_cols]))
    except ValueError: break
base = recs[0][0]
lo, hi = int(sys.argv[4]), int(sys.argv[5])
inside, cur, off = False, None, {}
for L in open(sys.argv[2]):
    if ".text." in L and L.strip().endswith(":"): inside = sys.argv[3] in L
    if not inside: continue
    m = re.search(r'File ".*ntt_ts.cu", line (\d+)', L)
    if m and int(m.group(1)) >= 176: cur = int(m.group(1))
    m = re.search(r'/\*([0-9a-f]{4,})\*/', L)
    if m and cur: off[int(m.group(1), 16)] = cur
src = open("/root/repo/paper_2212_14191_b200/csrc/ntt_ts.cu").read().split("\n")
c, ex, why = Counter(), Counter(), {}
for a, s, e, st in recs:
    ln = off.get(a - base, -1)
    if lo <= ln <= hi:
        c[ln] += s; ex[ln] += e
        w = why.setdefault(ln, Counter())
        for (_, h), v in zip(stall_cols, st): w[h] += v
tot = sum(c.values())
for ln, s in sorted(c.items()):
    if s * 200 < tot: continue
    top = ",".join(f"{h[6:]} {100*v/max(1,s):.0f}" for h, v in why[ln].most_common(3))
    print(f"{ln:4d} {100*s/tot:5.1f}% ex {ex[ln]:>10d} [{top}] {src[ln-1].strip()[:70]}")
