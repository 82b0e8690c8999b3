# batch-segmented operands (in-place repartition reads): full GPU suite + repart timings
cd $GRAFT_REPO_ROOT
OUT=gpurun_out/r02q
mkdir -p $OUT
for pr in bf16 fp32x3; do
  timeout 300 python tools/kernel_times.py bmm2_repart_p8_L1 5 $pr >> $OUT/times.txt 2>&1
  timeout 300 python tools/kernel_times.py bmm2_s_repart_p8_L1 5 $pr >> $OUT/times.txt 2>&1
done
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $OUT/pytest.log 2>&1
echo "pytest rc=$?" >> $OUT/pytest.log
echo done
