# ncu evidence of the current build: launch list of resident C3 steps (our
# kernels) and one --set full capture of k_step / k_forces.
#   gpurun -- 'bash tools/sess_ncu.sh TAG'
set -u
T=$1; O=gpurun_out/$T; mkdir -p $O
export SWF_HASH=0
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'^k_' -s 20 -c 60 --csv \
  --log-file $O/launches.csv python tools/kernel_times.py C3 4 > $O/launches_bench.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on \
  -k regex:'^k_(step|forces)(_list)?$' -s 8 -c 2 -o $O/prof \
  python tools/kernel_times.py C3 2 > $O/ncu_full.log 2>&1
echo done > $O/DONE
