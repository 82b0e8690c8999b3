cd $GRAFT_REPO_ROOT
for r in 1 2; do
for pl in hoc_p8_L1 ffnn_big_p8_L1 bmm2_p8_L1 chain3_p8_L1; do
  for sp in 2 0; do
    ED_GEMM_SERP=$sp timeout 300 python tools/kernel_times.py $pl 10 bf16 | sed "s/^/[serp=$sp] /"
  done
done
done
