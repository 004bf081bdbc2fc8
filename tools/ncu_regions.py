"""Summarise an ncu source-page CSV (SASS): executed instructions and stall
samples per 40-instruction window, with the dominant opcodes and stall
reasons (development aid).  usage: ncu_regions.py <src.csv> [window]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
win = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = rows[1]
iS = hdr.index("Warp Stall Sampling (All Samples)")
iE = hdr.index("Instructions Executed")
iSrc = hdr.index("Source")
stall_cols = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_") or "Stall" in h and "(" not in h]
recs = [r for r in rows[2:] if len(r) >= len(hdr)]
tot_e = sum(int(r[iE] or 0) for r in recs)
tot_s = sum(int(r[iS] or 0) for r in recs)
print(f"total executed {tot_e}  samples {tot_s}")
for i in range(0, len(recs), win):
    blk = recs[i:i + win]
    e = sum(int(b[iE] or 0) for b in blk)
    s = sum(int(b[iS] or 0) for b in blk)
    if e / max(tot_e, 1) < 0.01 and s / max(tot_s, 1) < 0.01:
        continue
    ops = {}
    for b in blk:
        t = b[iSrc].split()
        if not t:
            continue
        op = t[1] if t[0].startswith("@") and len(t) > 1 else t[0]
        op = op.split(".")[0]
        ops[op] = ops.get(op, 0) + 1
    top = sorted(ops.items(), key=lambda x: -x[1])[:6]
    print(f"{i:5d} exec {100 * e / tot_e:5.1f}% samp {100 * s / tot_s:5.1f}%  {top}")
