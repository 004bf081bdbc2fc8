bash tools/ab_perf.sh
TFHE_B200_LIB=$PWD/abtest/iss2.so timeout 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
rm -f gpurun_out/trace_*; TFHE_B200_LIB=$PWD/abtest/tr2.so timeout 300 python tools/prof_ntt.py 128
