#!/bin/bash
# key-switch epilogue iteration: parity (ckks + properties GPU tests) then HMULT timing
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ckks.py tests/test_gpu_properties.py -x -q > gpurun_out/gputest_ks.log 2>&1; echo "gputest rc=$?"; tail -2 gpurun_out/gputest_ks.log
for b in 32 128; do python tools/prof_hmult.py $b p_default fused; done
bash tools/kern_times.sh python tools/prof_hmult.py 32 p_default fused | head -4
