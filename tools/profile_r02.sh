#!/bin/bash
# Round-2 evidence run (one B200): bench line, per-kernel DRAM bytes of one
# N=2^16 NTT call (three-factor plan), launch list of the headline step, and
# full ncu captures of the two NTT pass kernels and the fused n=4096 kernel.
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_r02.json 2> gpurun_out/bench_r02.err
echo "bench rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file gpurun_out/ntt_dram.csv python tools/prof_ntt.py 128 \
  > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 1 --hmult-batch 0 \
  --set-a-batch 0 --hbm-kernels 0 --dnum5-batch 0 --sweep 0 --batch-sweep 0 --cpu-members 0 \
  > /dev/null 2>&1
for k in ntt_col_kernel ntt_row_kernel; do
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$k" -s 2 -c 1 -f \
    -o gpurun_out/$k python tools/prof_ntt.py 128 > gpurun_out/${k}_ncu.log 2>&1
  ncu -i gpurun_out/$k.ncu-rep --page details > gpurun_out/${k}_details.txt 2>/dev/null
  rm -f gpurun_out/$k.ncu-rep
done
bash tools/prof_fused.sh
echo done
