# r02h: producer lockstep experiment on the x3 kernel (DRAM traffic, time, parity)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r02h
ED_GEMM_SYNC=8,2 timeout 600 python -u -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -m gpu -q -x -k "fp32x3 or tensor_core" --timeout 300 > gpurun_out/r02h/pytest_sync.log 2>&1
for sy in none 8,2 8,4 16,2 4,4 32,2; do
  if [ "$sy" = none ]; then unset ED_GEMM_SYNC; else export ED_GEMM_SYNC=$sy; fi
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second --clock-control base -k regex:gemm -c 2 --csv --log-file gpurun_out/r02h/ncu_$sy.csv python tools/kernel_times.py hoc_p8_L1 1 fp32x3 > /dev/null 2>&1
  timeout 300 python tools/kernel_times.py hoc_p8_L1 5 fp32x3 >> gpurun_out/r02h/times_$sy.txt 2>&1
  timeout 300 python tools/kernel_times.py bmm2_p8_L1 5 fp32x3 >> gpurun_out/r02h/times_$sy.txt 2>&1
done
unset ED_GEMM_SYNC
echo done
