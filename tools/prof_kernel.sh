#!/bin/bash
# ncu --set full of one kernel (regex $1) of a python driver ($2...) into gpurun_out/<tag>_*
# usage: tools/prof_kernel.sh <tag> <kernel-regex> <skip> python tools/prof_X.py args
tag=$1; kre=$2; skip=$3; shift 3
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$kre" -s $skip -c 1 -f \
  -o gpurun_out/$tag "$@" > gpurun_out/${tag}_ncu.log 2>&1
ncu -i gpurun_out/$tag.ncu-rep --page details > gpurun_out/${tag}_details.txt
ncu -i gpurun_out/$tag.ncu-rep --page source --csv --print-source sass > gpurun_out/${tag}_src.csv
ncu -i gpurun_out/$tag.ncu-rep --page raw --csv > gpurun_out/${tag}_raw.csv
rm -f gpurun_out/$tag.ncu-rep
