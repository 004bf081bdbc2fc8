"""Per-kernel time shares of an ncu launch list
(`ncu --metrics gpu__time_duration.sum --csv --log-file X.csv ...`).

usage: python tools/ncu_launches.py X.csv [header-comment-lines...]
"""
import collections
import csv
import sys

rows = []
with open(sys.argv[1]) as fh:
    lines = [ln for ln in fh if ln.startswith('"')]
for r in csv.DictReader(lines):
    if r.get("Metric Name") == "gpu__time_duration.sum":
        v = float(r["Metric Value"].replace(",", ""))
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0,
                 "nsecond": 1e-6}.get(r["Metric Unit"], 1e-6)
        rows.append((r["Kernel Name"], v * scale))
agg = collections.defaultdict(lambda: [0.0, 0])
for name, ms in rows:
    short = name.split("(")[0][:100]
    agg[short][0] += ms
    agg[short][1] += 1
tot = sum(v[0] for v in agg.values())
for h in sys.argv[2:]:
    print("#", h)
print(f"# cold-cache serialised launches: compare SHARES, not absolutes")
print(f"# total {tot:.2f} ms over {len(rows)} launches")
for name, (ms, n) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f"{ms:10.3f} ms {100 * ms / tot:5.1f}%  n={n:5d}  avg={1e3 * ms / n:9.1f} us  {name}")
