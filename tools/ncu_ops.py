"""Executed-instruction histogram (per warp-element) of an ncu SASS source CSV.
usage: ncu_ops.py <src.csv> <elements processed by the kernel>"""
import csv, re, sys
from collections import Counter
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
iE, iS = hdr.index("Instructions Executed"), hdr.index("Source")
ops = Counter()
for r in rows[2:]:
    if len(r) < len(hdr):
        break
    try:
        e = int(r[iE])
    except ValueError:
        break
    s = re.sub(r"^@!?U?P\w+\s+", "", r[iS].strip())
    ops[s.split()[0] if s else "?"] += e
welem = float(sys.argv[2]) / 32
print("total per warp-element", sum(ops.values()) / welem)
heavy = ("IMAD", "IMAD.WIDE", "IMAD.WIDE.U32", "IMAD.HI.U32", "IMAD.MOV.U32", "IMAD.IADD",
         "IMAD.SHL.U32", "IMAD.U32", "HFMA2", "IMAD.X")
print("fmaheavy-class per warp-element", sum(v for k, v in ops.items() if k in heavy) / welem)
for op, v in ops.most_common(32):
    print(f"  {op:32s} {v / welem:6.2f}")
