#!/bin/bash
# split an ncu report's SASS source page per kernel launch: gpurun_out/<name>_k<i>.csv,
# dump the raw page and disassemble the current library for ncu_roles.py
name=$1
cd /root/repo/gpurun_out
ncu -i $name.ncu-rep --page source --csv --print-source sass > ${name}_src.csv 2>/dev/null
ncu -i $name.ncu-rep --page raw --csv > ${name}_raw.csv 2>/dev/null
awk -v n=$name 'BEGIN{k=0} /^"Kernel Name"/{k++} {print > (n "_k" k ".csv")}' ${name}_src.csv
rm -rf /tmp/cub && mkdir -p /tmp/cub && cd /tmp/cub && cuobjdump -xelf all /root/repo/paper_2212_14191_b200/libtfhe_b200.so >/dev/null
nvdisasm --print-line-info ntt_ts.sm_100a.cubin > /tmp/cub/ntt_ts.dis 2>/dev/null
ls /root/repo/gpurun_out/${name}_k*.csv
