set -u
O=gpurun_out/r3zq; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "region_loads or odd_sizes" > $O/pytest_region.log 2>&1; echo "exit $?" >> $O/pytest_region.log
timeout 900 python bench.py --config C5 --steps 20 --warmup 5 --e2e-steps 2 --no-cpu-baseline > $O/bench_c5.json 2> $O/bench_c5.err
timeout 900 python bench.py --config C4 > $O/bench_c4.json 2> $O/bench_c4.err
timeout 900 python bench.py --config C2 --no-cpu-baseline > $O/bench_c2.json 2> $O/bench_c2.err
timeout 600 paper_1705_00614_b200/swflood validate all > $O/validate.txt 2>&1; echo "exit $?" >> $O/validate.txt
echo done > $O/DONE
