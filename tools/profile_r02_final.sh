#!/bin/bash
# Round-2 final evidence run (one B200): both bench arms, the launch list of the
# headline step, DRAM bytes per NTT pass, and full ncu captures of the column
# pass, the grouped key-switch row pass (HMULT) and the base conversion.
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo "bench rc=$?"
python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
bash tools/ntt_traffic.sh
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_final.csv python bench.py --steps 2 --warmup 1 --hmult-batch 0 \
  --set-a-batch 0 --hbm-kernels 0 --dnum5-batch 0 --sweep 0 --batch-sweep 0 --cpu-members 0 \
  --cpu-numpy 0 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_hmult.csv python tools/prof_hmult.py 32 p_default fused > /dev/null 2>&1
cap() {  # tag kernel-regex skip cmd...
  tag=$1; re=$2; skip=$3; shift 3
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:$re" -s $skip -c 1 -f -o gpurun_out/$tag "$@" > gpurun_out/${tag}_ncu.log 2>&1
  ncu -i gpurun_out/$tag.ncu-rep --page details > gpurun_out/${tag}_details.txt 2>/dev/null
  ncu -i gpurun_out/$tag.ncu-rep --page raw --csv > gpurun_out/${tag}_raw.csv 2>/dev/null
  ncu -i gpurun_out/$tag.ncu-rep --page source --csv --print-source sass > gpurun_out/${tag}_src.csv 2>/dev/null
  rm -f gpurun_out/$tag.ncu-rep
}
cap col_final "col_kernel<.bool.0>" 1 python tools/prof_ntt.py 128
cap row_final "row_kernel<.int.0>" 1 python tools/prof_ntt.py 128
cap ksrow_final "row_kernel<.int.3>" 2 python tools/prof_hmult.py 32 p_default fused
cap bconv_final "bconv_tc" 2 python tools/prof_bconv.py 128
echo done
