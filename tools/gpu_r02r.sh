cd $GRAFT_REPO_ROOT
OUT=gpurun_out/r02r
mkdir -p $OUT
rm -f $OUT/times.txt
for pr in bf16 fp32x3; do
  timeout 300 python tools/kernel_times.py bmm2_repart_p8_L1 5 $pr >> $OUT/times.txt 2>&1
done
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "repart or fuzz or fullsize or parity" > $OUT/pytest.log 2>&1
echo "pytest rc=$?" >> $OUT/pytest.log
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:gemm python tools/kernel_times.py bmm2_repart_p8_L1 1 bf16 > $OUT/ncu.txt 2>&1
echo done
