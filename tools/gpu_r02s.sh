# bench lines of every config in both modes (no ncu), for the DESIGN tables
cd $GRAFT_REPO_ROOT
OUT=gpurun_out/r02s
mkdir -p $OUT
make -C oracle -s > /dev/null 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > $OUT/bench_default.jsonl 2> $OUT/bench_default.err
for c in hoc bmm2 bmm2_repart chain3 ffnn_big attn_big; do
  for pr in fp32x3 bf16; do
    timeout 600 python bench.py --config $c --precision $pr --extras '' --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 6 > $OUT/bench_${c}_$pr.jsonl 2>&1
  done
done
echo done
