#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over scripts/sanitize_run.py
# (every C-ABI entry point, C1-sized); logs in gpurun_out/sanitize_<tool>.log
set -u
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  extra=""
  [[ $tool == memcheck ]] && extra="--leak-check no"
  timeout 1500 compute-sanitizer --tool $tool $extra --target-processes all --print-limit 20 \
    python scripts/sanitize_run.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_$tool.log
done
grep -H "ERROR SUMMARY\|RACECHECK SUMMARY\|sanitize_run ok\|rc=" gpurun_out/sanitize_*.log
