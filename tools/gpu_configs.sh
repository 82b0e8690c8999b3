cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for c in chain3 hoc ffnn_big attn_big; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1; echo "rc=$?" >> gpurun_out/bench_$c.log
done
