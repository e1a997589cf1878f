# round-end evidence of the current build: GPU tests, smoke, the bench line,
# the reference arm, the FAST build's bench line
set -u
T=$1; O=gpurun_out/$T; mkdir -p $O
nvidia-smi > $O/nvidia-smi.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
timeout 300 python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench exit $?" >> $O/bench.err
timeout 900 python bench.py --impl reference > $O/reference.json 2> $O/reference.err
timeout 900 python bench.py --fast --no-cpu-baseline > $O/bench_fast.json 2> $O/bench_fast.err
echo done > $O/DONE
