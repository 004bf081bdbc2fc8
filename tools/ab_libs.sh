#!/bin/bash
# A/B the NTT and HMULT speed of alternative builds (abtest/*.so), interleaved
for rep in 1 2; do
  for lib in "$@"; do
    echo "== $lib (rep $rep)"
    TFHE_B200_LIB=$PWD/$lib timeout 300 python tools/quick_perf.py 2>&1 | head -1
    TFHE_B200_LIB=$PWD/$lib timeout 300 python tools/prof_hmult.py 32 2>&1 | tail -1
  done
done
