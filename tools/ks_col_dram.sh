timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:col_kernel --csv --log-file gpurun_out/kscol_dram.csv python tools/prof_hmult.py 128 p_default fused > /dev/null 2>&1
echo rc=$?
