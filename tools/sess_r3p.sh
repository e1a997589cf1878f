set -u
O=gpurun_out/r3p; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
timeout 900 python bench.py --config C4 --steps 20 --warmup 5 > $O/bench_c4.json 2> $O/bench_c4.err
timeout 900 python bench.py --config C5 --steps 20 --warmup 5 --e2e-steps 2 --no-cpu-baseline > $O/bench_c5.json 2> $O/bench_c5.err
echo done > $O/DONE
