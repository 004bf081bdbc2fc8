#!/bin/bash
# ncu --set full capture of the two TS NTT stages (N=2^16, 45 limbs, B=128) into gpurun_out/$1
name=${1:-ts_cur}
mkdir -p gpurun_out
timeout 800 ncu --set full --clock-control none --import-source on -k regex:ntt_ts -s 4 -c 2 -f \
  -o gpurun_out/$name python tools/prof_ntt.py 128 > gpurun_out/$name.log 2>&1
tail -2 gpurun_out/$name.log
