# r02e: multicast GEMM, exact exp, single-process multi-rank, split runtime: GPU suites + timings
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r02e
make -C oracle -s > gpurun_out/r02e/make.log 2>&1
./tools/micro/cluster_occ > gpurun_out/r02e/cluster_occ.txt 2>&1
timeout 900 python -u -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_generate.py -m gpu -q -x --timeout 300 > gpurun_out/r02e/pytest_parity.log 2>&1
timeout 900 python -u -m pytest tests/test_gpu_peer.py -m gpu -q --timeout 300 > gpurun_out/r02e/pytest_peer.log 2>&1
for mc in 0 1; do
  for c in hoc_p8_L1 bmm2_p8_L1 chain3_p8_L1 ffnn_big_p8_L1 attn_big_p8_L1; do
    for pr in bf16 fp32x3; do
      ED_GEMM_MC=$mc timeout 300 python tools/kernel_times.py $c 10 $pr >> gpurun_out/r02e/times_mc$mc.txt 2>&1
    done
  done
  for pr in fp32x3 bf16; do
    ED_GEMM_MC=$mc timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:gemm -c 2 --csv --log-file gpurun_out/r02e/ncu_hoc_mc${mc}_$pr.csv python tools/kernel_times.py hoc_p8_L1 1 $pr > /dev/null 2>&1
  done
done
for mc in 0 1; do
  ED_GEMM_MC=$mc timeout 600 python bench.py --extras '' --no-cpu-baseline --e2e-steps 1 > gpurun_out/r02e/bench_mc$mc.jsonl 2>&1
done
timeout 1500 python -u -m pytest tests/test_gpu_fullsize.py -m gpu -q -s --timeout 600 > gpurun_out/r02e/pytest_fullsize.log 2>&1
echo done
