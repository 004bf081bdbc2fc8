#!/bin/bash
# Re-entry check of HEAD on one B200: gpu tests, smoke, bench line, per-kernel times.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo "gputest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 600 bash tools/kern_times.sh python tools/prof_ntt.py 128 > gpurun_out/kt_ntt.txt 2>&1
timeout 600 bash tools/kern_times.sh python tools/prof_hmult.py 32 > gpurun_out/kt_hmult.txt 2>&1
tail -3 gpurun_out/gputest.log
echo done
