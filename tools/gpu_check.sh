cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/gpu_case.py gemm_nn_p1_L1 bf16 > gpurun_out/quick.log 2>&1
timeout 300 python tools/gpu_case.py gemm_ragged_p8_L1 bf16 >> gpurun_out/quick.log 2>&1
timeout 300 python tools/gpu_case.py gemm_tn_p8_L1 bf16 >> gpurun_out/quick.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/pytest.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "rc=$?" >> gpurun_out/bench.log
