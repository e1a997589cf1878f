# one --set full capture of k_step_list (source page) for the current build
#   gpurun -- 'bash tools/sess_ncu1.sh TAG'
set -u
T=$1; O=gpurun_out/$T; mkdir -p $O
export SWF_HASH=0
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:'^k_step_list$' -s 4 -c 1 -o $O/prof \
  python tools/kernel_times.py C3 2 > $O/ncu_full.log 2>&1
echo done > $O/DONE
