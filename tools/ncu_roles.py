"""Split ncu SASS stall samples of the TS NTT kernel by warp role.

usage: ncu_roles.py <ncu source csv (sass, one kernel)> <nvdisasm --print-line-info dump>
                    <mangled kernel substring> <role ranges "name:lo-hi,...">
Each SASS instruction is attributed to the last kernel-body line (of ntt_ts.cu,
outside the helper functions) that precedes it, then binned into the roles.
"""
import csv, os, re, sys
from collections import Counter
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
i_s, i_ex = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
stall_cols = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
recs = []
for r in rows[2:]:
    if len(r) < len(hdr): break
    try: recs.append((int(r[0], 16), int(r[i_s]), int(r[i_ex]), [int(r[i]) for i, _ in stall_cols]))
    except ValueError: break
base = recs[0][0]
fn = sys.argv[3]
roles = []
for part in sys.argv[4].split(","):
    name, rng = part.split(":")
    lo, hi = map(int, rng.split("-"))
    roles.append((name, lo, hi))
body_lo = min(r[1] for r in roles)
inside, cur, off2line = False, None, {}
for L in open(sys.argv[2]).read().split("\n"):
    if ".text." in L and L.strip().endswith(":"):
        inside = fn in L
    if not inside: continue
    m = re.search(r'File ".*' + re.escape(os.environ.get("SRC", "ntt_ts.cu")) + r'", line (\d+)', L)
    if m and int(m.group(1)) >= body_lo: cur = int(m.group(1))
    m = re.search(r'/\*([0-9a-f]{4,})\*/', L)
    if m and cur is not None: off2line[int(m.group(1), 16)] = cur
samp, exe, why = Counter(), Counter(), {}
for a, s, e, st in recs:
    ln = off2line.get(a - base, -1)
    role = next((n for n, lo, hi in roles if lo <= ln <= hi), "other")
    samp[role] += s; exe[role] += e
    w = why.setdefault(role, Counter())
    for (_, h), v in zip(stall_cols, st): w[h] += v
ts, te = sum(samp.values()), sum(exe.values())
for role in samp:
    top = ", ".join(f"{h[6:]} {100*v/max(1,samp[role]):.0f}%" for h, v in why[role].most_common(5))
    print(f"{role:10s} samples {100*samp[role]/ts:5.1f}%  exec {100*exe[role]/te:5.1f}% ({exe[role]})  [{top}]")

if len(sys.argv) > 5:
    # opcode histogram (executed warp instructions) for one role
    want = sys.argv[5]
    i_src = hdr.index("Source")
    ops = Counter()
    for r in rows[2:]:
        if len(r) < len(hdr): break
        try: a, e = int(r[0], 16), int(r[i_ex])
        except ValueError: break
        ln = off2line.get(a - base, -1)
        role = next((n for n, lo, hi in roles if lo <= ln <= hi), "other")
        if role != want: continue
        s = r[i_src].strip()
        s = re.sub(r"^@!?U?P\w+\s+", "", s)
        ops[s.split()[0] if s else "?"] += e
    tot = sum(ops.values())
    for op, v in ops.most_common(30):
        print(f"  {op:28s} {100*v/tot:5.1f}%  {v}")
