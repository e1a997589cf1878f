set -u
T=$1; O=gpurun_out/$T; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
shift
for L in default "$@"; do
  if [ "$L" = default ]; then timeout 300 python tools/kernel_times.py C3 10 >> $O/ab.jsonl 2>> $O/ab.err;
  else SWF_LIB=$L timeout 300 python tools/kernel_times.py C3 10 >> $O/ab.jsonl 2>> $O/ab.err; fi
done
SWF_HASH=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches.csv python tools/kernel_times.py C3 2 > /dev/null 2>&1
echo done > $O/DONE
