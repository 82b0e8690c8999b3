# bf16 GEMM: split-K code path removed from gemm_kernel (A/B against r02f's bench lines)
cd $GRAFT_REPO_ROOT
OUT=gpurun_out/r02ba
mkdir -p $OUT
make -C oracle -s > /dev/null 2>&1
for pl in chain3_p8_L1 bmm2_p8_L1 attn_big_p8_L1 ffnn_big_p8_L1 hoc_p8_L1; do
  KT_TOP=5 timeout 300 python tools/kernel_times.py $pl 10 bf16 >> $OUT/kt.txt 2>&1
done
cat $OUT/kt.txt
for c in chain3 bmm2 attn_big hoc; do
  timeout 600 python bench.py --config $c --precision bf16 --extras '' --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 6 > $OUT/bench_${c}_bf16.jsonl 2>&1
done
python tools/summarize_bench.py $OUT/bench_*.jsonl | cut -c1-200
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $OUT/pytest_gpu.txt 2>&1; tail -3 $OUT/pytest_gpu.txt
