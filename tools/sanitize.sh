#!/bin/bash
# compute-sanitizer over tools/sanitize_smoke.py (every kernel family, small
# shapes): memcheck, racecheck (shared memory) and synccheck.  Logs land in
# gpurun_out/sanitize_*.log; a summary line per tool is printed.
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 --target-processes all \
    python tools/sanitize_smoke.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|SANITIZE_SMOKE_OK|RACECHECK SUMMARY' gpurun_out/sanitize_$tool.log | tr '\n' ' ')"
done
