#!/bin/bash
# NTT (N=2^16, 45 limbs, B=128) under TFHE_DBG knobs of the debug build abtest/dbg.so
for k in 0 16 32 48 2 8192 8; do
  echo "== TFHE_DBG=$k"
  TFHE_DBG=$k TFHE_B200_LIB=$PWD/abtest/dbg.so timeout 300 python tools/quick_perf.py 2>&1 | head -2
done
