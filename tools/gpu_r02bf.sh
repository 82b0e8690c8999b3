# bf16 / tf32 tail split-K: A/B (ED_GEMM_SPLIT=0) on the configs with a partial last wave, then parity
cd $GRAFT_REPO_ROOT
OUT=gpurun_out/r02bf
mkdir -p $OUT
for r in 1 2; do
for c in chain3 attn_big ffnn_big bmm2; do
  for sp in 1 0; do
    ED_GEMM_SPLIT=$sp timeout 300 python bench.py --config $c --precision bf16 --extras '' --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$c split=$sp', d['ms_per_step'], d['value'], d['roofline']['frac'])" >> $OUT/ab.txt 2>&1
  done
  ED_GEMM_SPLIT=1 KT_TOP=6 timeout 300 python tools/kernel_times.py ${c}_p8_L1 5 bf16 >> $OUT/kt.txt 2>&1
  ED_GEMM_SPLIT=0 KT_TOP=6 timeout 300 python tools/kernel_times.py ${c}_p8_L1 5 bf16 >> $OUT/kt.txt 2>&1
done
done
cat $OUT/ab.txt $OUT/kt.txt
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fusion_fuzz.py tests/test_gpu_fuzz.py tests/test_gpu_fullsize.py -q -m gpu -x -p no:cacheprovider 2>&1 | tail -5
