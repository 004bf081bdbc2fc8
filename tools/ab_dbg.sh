#!/bin/bash
# time HMULT+rescale (P-Default, B=32) under TFHE_DBG knobs of the debug build abtest/dbg.so
for k in 0 2 8192 64 1 66 3; do
  echo "== TFHE_DBG=$k"
  TFHE_DBG=$k TFHE_B200_LIB=$PWD/abtest/dbg.so timeout 300 python tools/prof_hmult.py 32 2>&1 | tail -1
done
