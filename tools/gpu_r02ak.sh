# x3 tail split-K: parity, then A/B
cd $GRAFT_REPO_ROOT
make -C oracle -s > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -x -q -k "fp32x3 or x3" 2>&1 | tail -2
for r in 1 2; do
for pl in chain3_p8_L1 attn_big_p8_L1 ffnn_big_p8_L1 bmm2_p8_L1 hoc_p8_L1; do
  for sp in 1 0; do
    ED_GEMM_X3_SPLIT=$sp timeout 300 python tools/kernel_times.py $pl 10 fp32x3 | sed "s/^/[split=$sp] /"
  done
done
done
