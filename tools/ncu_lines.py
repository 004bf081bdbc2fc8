"""Aggregate ncu SASS-level samples / executed instructions per CUDA source line.

usage: ncu_lines.py <ncu source csv (sass)> <nvdisasm --print-line-info dump> <mangled kernel> [N] [source.cu]
"""
import csv, re, sys
from collections import Counter
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
i_a, i_s, i_ex = 0, hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
recs = []
for r in rows[2:]:
    if len(r) < len(hdr): break
    try: recs.append((int(r[0], 16), int(r[i_s]), int(r[i_ex])))
    except ValueError: break
base = recs[0][0]
# parse nvdisasm for the kernel
lines = open(sys.argv[2]).read().split("\n")
fn = sys.argv[3]
cur_line, inside, off2line = None, False, {}
for L in lines:
    if L.startswith(".text.") or ".text." in L and L.strip().endswith(":"):
        inside = fn in L
    if not inside: continue
    m = re.search(r'line (\d+)', L)
    if m and "//##" in L: cur_line = int(m.group(1))
    m = re.search(r'/\*([0-9a-f]{4,})\*/', L)
    if m and cur_line is not None: off2line[int(m.group(1), 16)] = cur_line
samp, exe = Counter(), Counter()
for a, s, e in recs:
    ln = off2line.get(a - base, -1)
    samp[ln] += s; exe[ln] += e
src = open(sys.argv[5] if len(sys.argv) > 5 else "paper_2212_14191_b200/csrc/ntt_ts.cu").read().split("\n")
tot = sum(samp.values()); tote = sum(exe.values())
N = int(sys.argv[4]) if len(sys.argv) > 4 else 30
print(f"total samples {tot}, executed {tote}")
for ln, s in samp.most_common(N):
    t = src[ln-1].strip()[:70] if 0 < ln <= len(src) else "?"
    print(f"line {ln:4d}  samp {100*s/tot:5.1f}%  exec {100*exe[ln]/tote:5.1f}%  {t}")
