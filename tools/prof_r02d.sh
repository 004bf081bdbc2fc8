#!/bin/bash
# full ncu of the grouped key-switch row pass (HMULT, P-Default B=32)
mkdir -p gpurun_out
k=ks_row3b
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:row_kernel<.int.3>" -s 2 -c 1 -f -o gpurun_out/$k python tools/prof_hmult.py 32 p_default fused > gpurun_out/${k}_ncu.log 2>&1
ncu -i gpurun_out/$k.ncu-rep --page details > gpurun_out/${k}_details.txt
ncu -i gpurun_out/$k.ncu-rep --page source --csv --print-source sass > gpurun_out/${k}_src.csv
ncu -i gpurun_out/$k.ncu-rep --page raw --csv > gpurun_out/${k}_raw.csv
rm -f gpurun_out/$k.ncu-rep
