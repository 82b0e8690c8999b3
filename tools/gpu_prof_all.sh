cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/prof
for c in bmm2 chain3 ffnn_big attn_big hoc; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/prof/bench_$c.jsonl 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/prof/launches_$c.csv python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
done
