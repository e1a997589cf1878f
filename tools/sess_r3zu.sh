set -u
O=gpurun_out/r3zu; mkdir -p $O
timeout 900 python bench.py --no-skip --no-cpu-baseline --steps 30 --warmup 5 --e2e-steps 3 > $O/bench_noskip.json 2> $O/bench_noskip.err
timeout 900 python bench.py --config C5W > $O/bench_c5w.json 2> $O/bench_c5w.err
timeout 900 python bench.py --gpus 2 --steps 20 --warmup 5 > $O/bench_g2.json 2> $O/bench_g2.err
echo done > $O/DONE
