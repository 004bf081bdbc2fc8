#!/bin/bash
# A/B of the limb-synchronous row-pass group order (TFHE_P3_STRIDED) on HMULT / HROTATE
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo "gputest rc=$?"; tail -2 gpurun_out/gputest.log
for s in 0 1; do
  for b in 32 128; do TFHE_P3_STRIDED=$s python tools/prof_hmult.py $b p_default fused; done
done
bash tools/kern_times.sh python tools/prof_hmult.py 32 p_default fused
