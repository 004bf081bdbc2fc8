#!/bin/bash
# base-conversion iteration: full GPU parity suite, then alpha=9 -> 54 timing at B = 8/32/128
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputest_bc.log 2>&1; echo "gputest rc=$?"; tail -3 gpurun_out/gputest_bc.log
for b in 8 32 128; do python tools/prof_bconv.py $b; done
python tools/prof_hmult.py 16 p_dnum5 fused
