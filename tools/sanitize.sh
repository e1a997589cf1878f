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
# the device free functions (forcing / block mask / sources) and the copyable
# stepper through the C++ drop-in (tests/native/free_api_test.cpp)
P=paper_1705_00614_b200
g++ -std=c++20 -O2 -I include tests/native/free_api_test.cpp -o /tmp/free_api_test -L $P \
  -lswflood_b200 -lswflood_cuda -Wl,-rpath,$PWD/$P && \
for tool in memcheck racecheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 --error-exitcode 9 \
    /tmp/free_api_test /tmp/free_api.bin > "$O/free_$tool.log" 2>&1
  echo "$tool exit $?" >> "$O/free_$tool.log"
done
