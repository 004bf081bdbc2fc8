#!/bin/bash
# N=2^12 NTT (2 limbs x 8192) under the resident kernel's TFHE_RES_DBG_VAL knobs (abtest/rdK.so):
# per-stage kernel durations from an ncu launch list
for lib in B rd256 rd512 rd2; do
  TFHE_B200_LIB=$PWD/abtest/$lib.so timeout 300 ncu --metrics gpu__time_duration.sum --csv --log-file gpurun_out/rdbg_$lib.csv python tools/prof_ntt_small.py 8192 > /dev/null 2>&1
  echo "== $lib: $(python tools/ncu_launches.py gpurun_out/rdbg_$lib.csv | grep ntt_res | awk '{print $NF, $6}' | tr '\n' ' ')"
done
