# r02g: promoted fp32x3 (multicast off by default): parity, full-size, timing vs chunk 0
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r02g
timeout 900 python -u -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -m gpu -q -x -k "fp32x3 or tensor_core" --timeout 300 > gpurun_out/r02g/pytest_x3.log 2>&1
for rep in 1 2; do
  for ch in 0 2 4; do
    for c in hoc_p8_L1 bmm2_p8_L1 chain3_p8_L1 ffnn_big_p8_L1; do
      ED_GEMM_X3_CHUNK=$ch timeout 300 python tools/kernel_times.py $c 3 fp32x3 >> gpurun_out/r02g/times.txt 2>&1
    done
    echo "-- chunk $ch" >> gpurun_out/r02g/times.txt
  done
done
timeout 1500 python -u -m pytest tests/test_gpu_fullsize.py -m gpu -q -s --timeout 600 -k "real_configs or integer_configs_fp32x3" > gpurun_out/r02g/pytest_fullsize.log 2>&1
timeout 600 python bench.py --extras '' --no-cpu-baseline --e2e-steps 1 > gpurun_out/r02g/bench.jsonl 2>&1
echo done
