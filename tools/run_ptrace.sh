#!/bin/bash
# column-pass timeline (TFHE_P3_TRACE build abtest/tr.so) + full ncu of both p3 passes
rm -f gpurun_out/ptrace_*
TFHE_B200_LIB=$PWD/abtest/tr.so timeout 300 python tools/ptrace_run.py
for f in gpurun_out/ptrace_*.bin; do echo "== $f"; python tools/ptrace_show.py $f 24; done
