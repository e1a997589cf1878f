#!/usr/bin/env bash
# One gpurun call: GPU tests, smoke, bench line, per-kernel times, ncu launch
# list and one ncu --set full capture of the two hot kernels.  Usage (here):
#   gpurun --timeout 2400 -- 'bash tools/gpu_session.sh TAG [skip-tests]'
set -u
TAG=${1:-r1}
SKIP_TESTS=${2:-}
O=gpurun_out/$TAG
mkdir -p "$O"
nvidia-smi > "$O/nvidia-smi.txt" 2>&1
lscpu > "$O/lscpu.txt" 2>&1
if [ -z "$SKIP_TESTS" ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q > "$O/pytest_gpu.log" 2>&1
  echo "pytest exit $?" >> "$O/pytest_gpu.log"
  timeout 300 python __graft_entry__.py smoke > "$O/smoke.log" 2>&1
  echo "smoke exit $?" >> "$O/smoke.log"
fi
timeout 900 python bench.py > "$O/bench.json" 2> "$O/bench.err"
echo "bench exit $?" >> "$O/bench.err"
timeout 900 python bench.py --impl reference > "$O/reference.json" 2> "$O/reference.err"
echo "reference exit $?" >> "$O/reference.err"
timeout 300 python tools/kernel_times.py C3 10 > "$O/kernel_times.json" 2>&1
# launch list of resident steps only (the e2e host-buffer steps are PCIe-bound
# and would distort the kernel shares)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file "$O/launches.csv" python tools/kernel_times.py C3 4 > "$O/launches_bench.log" 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:'^k_(step|forces)(_list)?$' -s 8 -c 2 -o "$O/prof" \
  python tools/kernel_times.py C3 2 > "$O/ncu_full.log" 2>&1
echo "done" > "$O/DONE"
