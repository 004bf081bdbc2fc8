#!/bin/bash
# A/B: time the N=2^16 NTT with several builds of the library (abtest/*.so)
for lib in abtest/*.so paper_2212_14191_b200/libtfhe_b200.so; do
  echo "== $lib"
  TFHE_B200_LIB=$PWD/$lib timeout 300 python tools/quick_perf.py 2>&1 | head -1
done
