# raster group size sweep (ED_GEMM_GROUP_M) on the power-capped fp32x3 configs, 20-step bench runs
cd $GRAFT_REPO_ROOT
OUT=gpurun_out/r02bb
mkdir -p $OUT
for rep in 1 2; do
for c in ffnn_big hoc; do
  for g in 8 16 4 32; do
    ED_GEMM_GROUP_M=$g timeout 600 python bench.py --config $c --precision fp32x3 --extras '' --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 1 > $OUT/bench_${c}_g${g}_r$rep.jsonl 2>&1
    echo "$c g=$g rep=$rep $(python tools/summarize_bench.py $OUT/bench_${c}_g${g}_r$rep.jsonl | cut -c1-150)"
  done
done
done
