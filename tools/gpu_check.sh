cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/pytest.log
for c in attn_big; do
timeout 600 python bench.py --config $c --steps 20 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1
done
