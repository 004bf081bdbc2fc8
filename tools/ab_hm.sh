#!/bin/bash
# A/B the fused P-Default HMULT+rescale (B=32) between builds: LIBS="a.so b.so" bash tools/ab_hm.sh
for rep in 1 2; do for lib in ${LIBS}; do
  echo "== $lib"; TFHE_B200_LIB=$PWD/$lib timeout 300 python tools/prof_hmult.py 32 p_default fused 2>&1 | tail -1
done; done
