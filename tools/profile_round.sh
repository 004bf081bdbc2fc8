#!/bin/bash
# Round profiling pass on ONE GPU (run under gpurun from the repo root):
#   1. launch list of the bench command (gpu__time_duration per launch, cold, serialised)
#   2. ncu --set full of the two TS NTT stage kernels at the bench shape
#   3. ncu --set full of one HMULT+rescale pipeline (every kernel once) at P-Default
# Outputs land in gpurun_out/<tag>_*; summarise with tools/ncu_summary.py / ncu_launches.py.
tag=${1:-r01}
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
  --log-file gpurun_out/${tag}_launches.csv \
  python bench.py --steps 2 --warmup 1 --hmult-batch 4 --cpu-members 0 > gpurun_out/${tag}_launches_bench.log 2>&1
echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ntt_ts -s 4 -c 2 -f \
  -o gpurun_out/${tag}_ntt_ts python tools/prof_ntt.py 128 > gpurun_out/${tag}_ntt_ts.log 2>&1
echo "ntt_ts full rc=$?"
ncu -i gpurun_out/${tag}_ntt_ts.ncu-rep --page raw --csv > gpurun_out/${tag}_ntt_ts_raw.csv 2>/dev/null
ncu -i gpurun_out/${tag}_ntt_ts.ncu-rep --page details > gpurun_out/${tag}_ntt_ts_details.txt 2>/dev/null
if [ "${2:-}" = "hmult" ]; then
  timeout 900 ncu --set full --clock-control none -s 60 -c 40 -f \
    -o gpurun_out/${tag}_hmult python tools/prof_hmult.py 8 > gpurun_out/${tag}_hmult.log 2>&1
  echo "hmult full rc=$?"
  ncu -i gpurun_out/${tag}_hmult.ncu-rep --page raw --csv > gpurun_out/${tag}_hmult_raw.csv 2>/dev/null
fi
# keep the merged-back gpurun_out/ under 64 MiB: exports only, reports dropped
ncu -i gpurun_out/${tag}_ntt_ts.ncu-rep --page source --csv --print-source sass > gpurun_out/${tag}_ntt_ts_src.csv 2>/dev/null
rm -f gpurun_out/*.ncu-rep
gzip -f gpurun_out/${tag}_*_src.csv
du -sh gpurun_out
