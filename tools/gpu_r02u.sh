# lo shadows written by their producers (x3 GEMM epilogue, softmax, refinement folds): suite + fp32x3 configs
cd $GRAFT_REPO_ROOT
OUT=gpurun_out/r02u
mkdir -p $OUT
make -C oracle -s > /dev/null 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.txt
tail -3 $OUT/pytest_gpu.txt
for c in bmm2 bmm2_repart chain3 ffnn_big attn_big; do
  timeout 600 python bench.py --config $c --precision fp32x3 --extras '' --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 > $OUT/bench_${c}.jsonl 2>&1
  python - $OUT/bench_${c}.jsonl <<'PY'
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d=json.loads(l); print(d['config']['graph'], d['value'], d['ms_per_step'], [(k['name'],k['launches'],round(k['ms'],3)) for k in d['roofline']['kernels']])
PY
done
