cd $GRAFT_REPO_ROOT
for prec in tf32 bf16; do
for c in gemm_nn_p1_L1 gemm_tn_p1_L1 gemm_nt_p1_L1 gemm_swap_p1_L1 gemm_ragged_p1_L1 gemm_batch_p1_L1 gemm_heads_p1_L1 gemm_merge_p1_L1 gemm_nn_p8_L1 gemm_merge_p8_L1 matmul_p1_L1 attention_p1_L1 ffnn_p1_L1; do
  timeout 120 python tools/gpu_case.py $c $prec >> gpurun_out/debug.log 2>&1 || echo "FAIL $c $prec rc=$?" >> gpurun_out/debug.log
done; done
timeout 300 compute-sanitizer --tool memcheck python tools/gpu_case.py attention_p1_L1 bf16 > gpurun_out/sanitizer.log 2>&1
