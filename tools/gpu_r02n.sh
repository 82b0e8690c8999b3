# GEMM warp-wide issue: full GPU suite + per-launch times of every config in both modes
cd $GRAFT_REPO_ROOT
OUT=gpurun_out/r02n
mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $OUT/pytest.log 2>&1
echo "pytest rc=$?" >> $OUT/pytest.log
for c in hoc bmm2 bmm2_repart chain3 ffnn_big attn_big; do
  for pr in bf16 fp32x3; do
    timeout 300 python tools/kernel_times.py ${c}_p8_L1 5 $pr >> $OUT/times.txt 2>&1
  done
done
echo done
