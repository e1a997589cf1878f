set -u
O=gpurun_out/r3f; mkdir -p $O
for L in paper_1705_00614_b200/variants/libswf_fastA.so paper_1705_00614_b200/variants/libswf_fastB.so paper_1705_00614_b200/libswflood_cuda_fast.so; do
  SWF_LIB=$L timeout 300 python tools/dbg_fast.py c3_crop 40 0.0 >> $O/dbg.txt 2>&1
done
timeout 300 python tools/kernel_times.py C3 10 >> $O/ab.jsonl 2>> $O/ab.err
SWF_LIB=paper_1705_00614_b200/variants/libswf_fused.so timeout 300 python tools/kernel_times.py C3 10 >> $O/ab.jsonl 2>> $O/ab.err
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
echo done > $O/DONE
