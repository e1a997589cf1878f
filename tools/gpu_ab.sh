#!/usr/bin/env bash
# A/B per-kernel times of library variants on C3 (+ the GPU parity suite).
#   gpurun -- 'bash tools/gpu_ab.sh TAG [tests] lib1.so lib2.so ...'
set -u
TAG=$1; shift
O=gpurun_out/$TAG; mkdir -p "$O"
if [ "${1:-}" = "tests" ]; then
  shift
  timeout 1200 python -m pytest tests -m gpu -x -q > "$O/pytest_gpu.log" 2>&1
  echo "pytest exit $?" >> "$O/pytest_gpu.log"
fi
timeout 300 python tools/kernel_times.py C3 10 >> "$O/ab.jsonl" 2>> "$O/ab.err"
for L in "$@"; do
  SWF_LIB=$L timeout 300 python tools/kernel_times.py C3 10 >> "$O/ab.jsonl" 2>> "$O/ab.err"
done
timeout 300 python tools/kernel_times.py C3 10 >> "$O/ab.jsonl" 2>> "$O/ab.err"
