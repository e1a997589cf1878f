set -u
O=gpurun_out/r3zzb; mkdir -p $O
V=paper_1705_00614_b200/variants
for L in default $V/libswf_unr2.so $V/libswf_fmin8.so default $V/libswf_unr2.so $V/libswf_fmin8.so; do
  if [ $L = default ]; then python tools/kernel_times.py C3 10; else SWF_LIB=$L python tools/kernel_times.py C3 10; fi
done > $O/ab.jsonl 2>&1
echo done > $O/DONE
