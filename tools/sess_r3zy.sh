set -u
O=gpurun_out/r3zy; mkdir -p $O
timeout 900 python bench.py --config C5W --no-skip --no-cpu-baseline --steps 30 --warmup 5 --e2e-steps 3 > $O/bench_c5w_noskip.json 2> $O/bench_c5w_noskip.err
timeout 900 python bench.py --config C5 --no-skip --no-cpu-baseline --steps 10 --warmup 3 --e2e-steps 2 > $O/bench_c5_noskip.json 2> $O/bench_c5_noskip.err
echo done > $O/DONE
