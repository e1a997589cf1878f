set -u
O=gpurun_out/r3zo; mkdir -p $O
V=paper_1705_00614_b200/variants
for L in default $V/libswf_nopf.so default $V/libswf_nopf.so; do
  if [ $L = default ]; then python tools/kernel_times.py C3 10; else SWF_LIB=$L python tools/kernel_times.py C3 10; fi
done > $O/ab.jsonl 2>&1
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
echo done > $O/DONE
