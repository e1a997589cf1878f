set -u
O=gpurun_out/r3i; mkdir -p $O
SWF_HASH=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_x" -c 6 --csv --log-file $O/launches.csv python tools/kernel_times.py C3 2 > /dev/null 2>&1
timeout 300 python tools/kernel_times.py C3 10 >> $O/ab.jsonl 2>> $O/ab.err
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
echo done > $O/DONE
