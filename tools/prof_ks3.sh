timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:ntt_ts_kernel<.int.2, .int.256, .int.3>' -s 2 -c 1 -f -o gpurun_out/ks3 python tools/prof_hmult.py 8 > gpurun_out/ks3_ncu.log 2>&1
ncu -i gpurun_out/ks3.ncu-rep --page details > gpurun_out/ks3_details.txt
ncu -i gpurun_out/ks3.ncu-rep --page source --csv --print-source sass > gpurun_out/ks3_src.csv
ncu -i gpurun_out/ks3.ncu-rep --page raw --csv > gpurun_out/ks3_raw.csv
rm -f gpurun_out/ks3.ncu-rep
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:ntt_ts_kernel<.int.2, .int.256, .int.0>' -s 2 -c 1 -f -o gpurun_out/ks0 python tools/prof_ntt.py 128 > gpurun_out/ks0_ncu.log 2>&1
ncu -i gpurun_out/ks0.ncu-rep --page details > gpurun_out/ks0_details.txt
ncu -i gpurun_out/ks0.ncu-rep --page source --csv --print-source sass > gpurun_out/ks0_src.csv
rm -f gpurun_out/ks0.ncu-rep
