#!/bin/bash
# DRAM bytes per launch of both N=2^16 NTT passes at the bench shape (B=128, 45 limbs):
# gpurun_out/ntt_dram.csv -> profiles/ntt_dram_traffic.json (tools/ntt_traffic_json.py)
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file gpurun_out/ntt_dram.csv python tools/prof_ntt.py 128 \
  > /dev/null 2>&1
echo "ncu rc=$?"
