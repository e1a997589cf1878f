set -u
O=gpurun_out/r3c; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench exit $?" >> $O/bench.err
timeout 900 python bench.py --impl reference > $O/reference.json 2> $O/reference.err; echo "ref exit $?" >> $O/reference.err
echo done > $O/DONE
