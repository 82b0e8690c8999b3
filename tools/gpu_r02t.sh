# re-entry check: GPU suite, smoke, default bench line on the restored HEAD
cd $GRAFT_REPO_ROOT
OUT=gpurun_out/r02t
mkdir -p $OUT
make -C oracle -s > /dev/null 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1
timeout 900 python bench.py > $OUT/bench_default.jsonl 2> $OUT/bench_default.err
tail -3 $OUT/pytest_gpu.txt; cat $OUT/bench_default.jsonl | head -c 3000
