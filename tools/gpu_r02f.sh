# r02f: fp32x3 with promoted accumulation — accuracy vs chunk size, parity, timing
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r02f
for ch in 0 1 2 4 8; do
  echo "== chunk $ch" >> gpurun_out/r02f/kprobe.txt
  ED_GEMM_X3_CHUNK=$ch timeout 300 python tools/x3_kprobe.py >> gpurun_out/r02f/kprobe.txt 2>&1
  ED_GEMM_X3_CHUNK=$ch timeout 300 python tools/kernel_times.py hoc_p8_L1 5 fp32x3 >> gpurun_out/r02f/times.txt 2>&1
  ED_GEMM_X3_CHUNK=$ch timeout 300 python tools/kernel_times.py bmm2_p8_L1 5 fp32x3 >> gpurun_out/r02f/times.txt 2>&1
  ED_GEMM_X3_CHUNK=$ch timeout 300 python tools/kernel_times.py chain3_p8_L1 5 fp32x3 >> gpurun_out/r02f/times.txt 2>&1
  echo "-- chunk $ch" >> gpurun_out/r02f/times.txt
done
timeout 900 python -u -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -m gpu -q -x -k "fp32x3 or tensor_core" --timeout 300 > gpurun_out/r02f/pytest_x3.log 2>&1
timeout 600 python bench.py --extras '' --no-cpu-baseline --e2e-steps 1 > gpurun_out/r02f/bench.jsonl 2>&1
timeout 1500 python -u -m pytest tests/test_gpu_fullsize.py -m gpu -q -s --timeout 600 -k "real_configs or integer_configs_fp32x3" > gpurun_out/r02f/pytest_fullsize.log 2>&1
echo done
