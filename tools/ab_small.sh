#!/bin/bash
# A/B of the small-n NTT and Set_A / Set_B HMULT(+rescale) between builds (LIBS, default
# abtest/A.so abtest/B.so), interleaved
for rep in 1 2; do for lib in ${LIBS:-abtest/A.so abtest/B.so}; do echo "== $lib"
TFHE_B200_LIB=$PWD/$lib timeout 300 python tools/prof_ntt_small.py 8192 2>&1 | tail -1
TFHE_B200_LIB=$PWD/$lib timeout 300 python tools/prof_ntt_small.py 8192 8192 2>&1 | tail -1
TFHE_B200_LIB=$PWD/$lib timeout 300 python tools/prof_hmult.py 4096 set_a 2>&1 | tail -1
TFHE_B200_LIB=$PWD/$lib timeout 300 python tools/prof_hmult.py 4096 set_a fused 2>&1 | tail -1
TFHE_B200_LIB=$PWD/$lib timeout 300 python tools/prof_hmult.py 1024 set_b fused 2>&1 | tail -1
done; done
