set -u
O=gpurun_out/${1:-ncu}; mkdir -p $O
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file "$O/launches.csv" python tools/kernel_times.py C3 4 > "$O/launches_bench.log" 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:'^k_(step|forces)(_list)?$' -s 8 -c 2 -o "$O/prof" \
  python tools/kernel_times.py C3 2 > "$O/ncu_full.log" 2>&1
