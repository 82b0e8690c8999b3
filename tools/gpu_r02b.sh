# r02b: fused x3 GEMM stage — parity (fp32x3 tests) + bench lines
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r02b
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -m gpu -q -x -k "fp32x3" --timeout 600 > gpurun_out/r02b/pytest_x3.log 2>&1
for c in hoc bmm2 bmm2_repart chain3; do
  timeout 600 python bench.py --config $c --precision fp32x3 --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/r02b/bench_${c}_fp32x3.jsonl 2>&1
done
timeout 600 python bench.py --config hoc --precision fp32x3 --steps 100 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/r02b/bench_hoc_fp32x3_100.jsonl 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second --clock-control none --csv --log-file gpurun_out/r02b/launches_hoc.csv python bench.py --config hoc --precision fp32x3 --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
echo done
