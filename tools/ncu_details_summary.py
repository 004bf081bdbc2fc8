"""Condense an `ncu --page details` text export to one "[section] metric value
unit" line per metric and kernel (drops the advisory prose).

usage: python tools/ncu_details_summary.py details.txt [header lines...]
"""
import re
import sys

lines = open(sys.argv[1]).read().splitlines()
for h in sys.argv[2:]:
    print("#", h)
section = ""
for ln in lines:
    m = re.match(r"^  (\S.*\(\d+, \d+, \d+\)x\(\d+, \d+, \d+\).*)$", ln)
    if m:
        print("\n== " + m.group(1).split(" (")[0])
        continue
    m = re.match(r"^\s+Section: (.*)$", ln)
    if m:
        section = m.group(1)[:28]
        continue
    m = re.match(r"^\s{4}(\S[\w /().%-]*?)\s{2,}(\S+)?\s+([\d.,]+)\s*$", ln)
    if m and not ln.strip().startswith(("-", "Metric Name")):
        name, unit, val = m.group(1).strip(), (m.group(2) or ""), m.group(3)
        print(f"  [{section:28s}] {name:52s} {val:>14s} {unit}")
