# serpentine K in the x3 GEMM: A/B (kernel times, DRAM bytes), integer full-size parity
cd $GRAFT_REPO_ROOT
make -C oracle -s > /dev/null 2>&1
for r in 1 2; do
for pl in hoc_p8_L1 ffnn_big_p8_L1 bmm2_p8_L1; do
  for sp in 1 0; do
    ED_GEMM_SERP=$sp timeout 300 python tools/kernel_times.py $pl 5 fp32x3 | sed "s/^/[serp=$sp] /"
  done
done
done
for sp in 1 0; do
  ED_GEMM_SERP=$sp timeout 600 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none -k regex:gemm_x3 -c 2 python tools/kernel_times.py hoc_p8_L1 1 fp32x3 2>/dev/null | grep -E "dram__bytes_read|gpu__time" | sed "s/^/[serp=$sp] /"
done
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -k "integer_configs_fp32x3" 2>&1 | tail -1
