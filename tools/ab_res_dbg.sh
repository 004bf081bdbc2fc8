#!/bin/bash
# N=2^12 NTT (2 limbs x 8192) per-stage kernel times (ncu launch list) under the
# resident kernel's timing probes: abtest/rdK.so built with -DTFHE_RES_DBG_VAL=K
# (see ntt_tc.cu), abtest/B.so the normal build
for lib in B rd1 rd2 rd512 rd4 rd8; do
  [ -f abtest/$lib.so ] || continue
  TFHE_B200_LIB=$PWD/abtest/$lib.so timeout 300 ncu --metrics gpu__time_duration.sum --csv \
    --log-file gpurun_out/rdbg_$lib.csv python tools/prof_ntt_small.py 8192 > /dev/null 2>&1
  echo "== $lib"; python tools/ncu_launches.py gpurun_out/rdbg_$lib.csv | grep ntt_res | cut -c1-110
done
