cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for c in bmm2 hoc chain3; do
timeout 600 python bench.py --config $c --steps 30 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1
done
