"""gpurun_out/ntt_dram.csv (tools/ntt_traffic.sh) -> profiles/ntt_dram_traffic.json:
average DRAM bytes and duration per launch of each N=2^16 NTT pass kernel
(ncu, --clock-control none, cold caches, serialised launches)."""
import collections
import csv
import json
import sys

N, L, B = 1 << 16, 45, 128
rows = collections.defaultdict(lambda: collections.defaultdict(list))
src = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/ntt_dram.csv"
for r in csv.DictReader(l for l in open(src) if not l.startswith("==")):
    k = r["Kernel Name"]
    if "ntt_col_kernel" not in k and "ntt_row_kernel" not in k:
        continue
    v = float(r["Metric Value"].replace(",", ""))
    unit = r.get("Metric Unit", "")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-6, "ns": 1e-6,
             "us": 1e-3, "ms": 1.0,
             "usecond": 1e-3, "msecond": 1.0}.get(unit, 1)
    rows[k.split("(")[0]][r["Metric Name"]].append(v * scale)
launches = []
for k, m in sorted(rows.items()):
    avg = lambda key: sum(m[key]) / len(m[key])  # noqa: E731
    launches.append({"kernel": k, "launches": len(m["gpu__time_duration.sum"]),
                     "dram_read_bytes": avg("dram__bytes_read.sum"),
                     "dram_write_bytes": avg("dram__bytes_write.sum"),
                     "duration_ms": avg("gpu__time_duration.sum")})
fwd = [r for r in launches if "<0>" in r["kernel"] or "(bool)0" in r["kernel"] or "false" in r["kernel"]]
out = {"batch": B, "limbs": L, "N": N, "transform_plan": [32, 32, 64],
       "source": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                 "--clock-control none on tools/prof_ntt.py 128 (2 x forward + inverse NTT call, "
                 "each = ntt_col_kernel + ntt_row_kernel); tools/ntt_traffic.sh",
       "launches": launches,
       "algorithmic_bytes_per_launch": 8 * N * L * B,
       "compulsory_bytes_per_ntt_call": 8 * N * L * B,
       "design_bytes_per_ntt_call": 16 * N * L * B}
col = [r for r in launches if "col_kernel" in r["kernel"]]
row = [r for r in launches if "row_kernel" in r["kernel"]]
if col and row:
    per = lambda rs: sum(r["dram_read_bytes"] + r["dram_write_bytes"] for r in rs) / len(rs)  # noqa
    out["bytes_per_ntt_call"] = per(col) + per(row)
json.dump(out, open("profiles/ntt_dram_traffic.json", "w"), indent=1)
print(json.dumps(out, indent=1))
