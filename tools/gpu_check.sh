cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/pytest.log
for c in attn_big ffnn_big bmm2 hoc; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1; echo "rc=$?" >> gpurun_out/bench_$c.log
done
