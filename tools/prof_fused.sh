#!/bin/bash
# ncu full capture (source-level) of the fused n=4096 NTT kernel
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:ntt_fused" -s 3 -c 1 -f \
  -o gpurun_out/fused python tools/perf_small.py > gpurun_out/fused_ncu.log 2>&1
ncu -i gpurun_out/fused.ncu-rep --page details > gpurun_out/fused_details.txt
ncu -i gpurun_out/fused.ncu-rep --page source --csv --print-source sass > gpurun_out/fused_src.csv
ncu -i gpurun_out/fused.ncu-rep --page raw --csv > gpurun_out/fused_raw.csv
rm -f gpurun_out/fused.ncu-rep
