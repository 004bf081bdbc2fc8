#!/bin/bash
# per-kernel average durations (ncu gpu__time_duration, cold/serialised) of a
# driver for each lib: LIBS="a.so b.so" bash tools/kern_times.sh python tools/prof_ntt.py 128
for lib in ${LIBS:-paper_2212_14191_b200/libtfhe_b200.so}; do
  echo "== $lib"
  TFHE_B200_LIB=$PWD/$lib timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none \
    --csv --log-file /tmp/kt.csv "$@" > /dev/null 2>&1
  python - <<'PY'
import csv, collections
d = collections.defaultdict(list)
for r in csv.DictReader(l for l in open('/tmp/kt.csv') if not l.startswith('==')):
    if r.get('Metric Name') == 'gpu__time_duration.sum':
        d[r['Kernel Name'].split('(')[0][-60:]].append(float(r['Metric Value'].replace(',', '')))
for k, v in sorted(d.items(), key=lambda x: -sum(x[1])):
    print(f"  {k:60s} n={len(v):4d} avg={sum(v)/len(v)/1e3:9.1f} us  total={sum(v)/1e6:8.3f} ms")
PY
done
