set -u
O=gpurun_out/r3d; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_fast.py -q -p no:cacheprovider > $O/pytest_fast.log 2>&1; echo "exit $?" >> $O/pytest_fast.log
timeout 300 python tools/kernel_times.py C3 10 >> $O/ab.jsonl 2>> $O/ab.err
SWF_FLAVOR=fast timeout 300 python tools/kernel_times.py C3 10 >> $O/ab.jsonl 2>> $O/ab.err
timeout 900 python bench.py --fast --no-cpu-baseline > $O/bench_fast.json 2> $O/bench_fast.err
echo done > $O/DONE
