# ncu launch list (our kernels only) + one --set full capture of the given kernels.
#   bash tools/ncu_kernels.sh TAG 'regex' [SWF_LIB]
set -u
T=$1; RX=$2; O=gpurun_out/$T; mkdir -p $O
[ -n "${3:-}" ] && export SWF_LIB=$3
export SWF_HASH=0
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'^k_' -c 40 --csv --log-file $O/launches.csv python tools/kernel_times.py C3 2 > $O/launches.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"$RX" -s 4 -c 2 -o $O/prof python tools/kernel_times.py C3 2 > $O/ncu_full.log 2>&1
echo done > $O/DONE
