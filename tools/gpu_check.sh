cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -x -p no:cacheprovider -k "attn" > gpurun_out/pytest_attn.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_attn.log
timeout 600 python bench.py --config attn_big --steps 20 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/bench_attn.log 2>&1; echo "rc=$?" >> gpurun_out/bench_attn.log
