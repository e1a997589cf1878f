set -u
O=gpurun_out/r3a; mkdir -p $O
nvidia-smi > $O/nvidia-smi.txt 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o /tmp/fp64_peak tools/fp64_peak.cu && timeout 120 /tmp/fp64_peak > $O/fp64_peak.json 2> $O/fp64_peak.err
timeout 300 python tools/kernel_times.py C3 10 > $O/kt.json 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
echo done > $O/DONE
