#!/bin/bash
# A/B the N=2^16 NTT (fwd / inv, B=128 x 45 limbs) and P-Default HMULT+rescale between
# builds: LIBS="abtest/a.so abtest/b.so" bash tools/ab_n16.sh
for rep in 1 2; do for lib in ${LIBS:-abtest/base.so paper_2212_14191_b200/libtfhe_b200.so}; do
  echo "== $lib"
  TFHE_B200_LIB=$PWD/$lib timeout 300 python tools/perf_n16.py 128 2>&1 | tail -2
  [ -n "$HM" ] && TFHE_B200_LIB=$PWD/$lib timeout 300 python tools/prof_hmult.py 32 2>&1 | tail -1
done; done
