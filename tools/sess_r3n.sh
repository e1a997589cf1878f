set -u
O=gpurun_out/r3n; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
timeout 300 python tools/kernel_times.py C3 10 >> $O/ab.jsonl 2>> $O/ab.err
echo done > $O/DONE
