# r02i: producer lockstep on by default for every GEMM: GPU suite, timings on/off, DRAM
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r02i
make -C oracle -s > /dev/null 2>&1
timeout 1200 python -u -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/r02i/pytest_gpu.log 2>&1
for sy in 0,0 16,2; do
  export ED_GEMM_SYNC=$sy
  for c in hoc_p8_L1 bmm2_p8_L1 chain3_p8_L1 ffnn_big_p8_L1 attn_big_p8_L1 bmm2_repart_p8_L1; do
    for pr in bf16 fp32x3; do
      timeout 300 python tools/kernel_times.py $c 5 $pr >> gpurun_out/r02i/times_$sy.txt 2>&1
    done
  done
  for pr in bf16 fp32x3; do
    timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:gemm --csv --log-file gpurun_out/r02i/ncu_${sy}_hoc_$pr.csv python tools/kernel_times.py hoc_p8_L1 1 $pr > /dev/null 2>&1
    timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:gemm --csv --log-file gpurun_out/r02i/ncu_${sy}_ffnn_$pr.csv python tools/kernel_times.py ffnn_big_p8_L1 1 $pr > /dev/null 2>&1
  done
done
unset ED_GEMM_SYNC
timeout 600 python bench.py > gpurun_out/r02i/bench_default.jsonl 2> gpurun_out/r02i/bench_default.err
echo done
