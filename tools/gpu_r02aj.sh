cd $GRAFT_REPO_ROOT
for r in 1 2; do
for pl in chain3_p8_L1 attn_big_p8_L1 bmm2_p8_L1; do
  for bn in 256 128; do
    ED_GEMM_BN=$bn timeout 300 python tools/kernel_times.py $pl 10 fp32x3 | sed "s/^/[bn=$bn] /"
  done
done
done
