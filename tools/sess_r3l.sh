set -u
O=gpurun_out/r3l; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_multidevice.py -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
timeout 900 python bench.py --gpus 2 --steps 20 --warmup 5 --e2e-steps 1 > $O/bench2.json 2> $O/bench2.err; echo "exit $?" >> $O/bench2.err
echo done > $O/DONE
