set -u
O=gpurun_out/r3zza; mkdir -p $O
V=paper_1705_00614_b200/variants
for L in default $V/libswf_l2p0.so $V/libswf_l2p2.so default $V/libswf_l2p0.so $V/libswf_l2p2.so; do
  if [ $L = default ]; then python tools/kernel_times.py C3 10; else SWF_LIB=$L python tools/kernel_times.py C3 10; fi
done > $O/ab.jsonl 2>&1
echo done > $O/DONE
