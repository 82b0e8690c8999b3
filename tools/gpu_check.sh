cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/quick.log
for c in gemm_nn_p1_L1 gemm_tn_p1_L1 gemm_batch_p8_L1 gemm_nn_p8_L1 matmul_p1_L1; do timeout 120 python tools/gpu_case.py $c tf32 >> gpurun_out/quick.log 2>&1; done
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/pytest.log
