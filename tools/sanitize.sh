#!/usr/bin/env bash
# compute-sanitizer over tools/sanitize_run.py:
#   gpurun -- 'bash tools/sanitize.sh TAG'
set -u
O=gpurun_out/${1:-sanitize}; mkdir -p "$O"
timeout 600 python tools/sanitize_run.py > "$O/plain.log" 2>&1; echo "plain exit $?" >> "$O/plain.log"
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 --error-exitcode 9 \
    python tools/sanitize_run.py > "$O/$tool.log" 2>&1
  echo "$tool exit $?" >> "$O/$tool.log"
done
