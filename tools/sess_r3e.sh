set -u
O=gpurun_out/r3e; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
echo done > $O/DONE
