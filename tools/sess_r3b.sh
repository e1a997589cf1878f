set -u
O=gpurun_out/r3b; mkdir -p $O
nvidia-smi > $O/nvidia-smi.txt 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_peak tools/fp64_peak.cu && timeout 120 /tmp/fp64_peak > $O/fp64_peak.json 2> $O/fp64_peak.err
bash tools/gpu_session.sh r3b
