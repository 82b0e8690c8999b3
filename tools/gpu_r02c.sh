# r02c: new bench.py default line; raster group sweep (DRAM bytes) on hoc fp32x3 / bf16
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r02c
timeout 900 python bench.py > gpurun_out/r02c/bench_default.jsonl 2> gpurun_out/r02c/bench_default.err
for gm in 2 4 8 16 32; do
  for pr in fp32x3 bf16; do
    ED_GEMM_GROUP_M=$gm timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second --clock-control base -k regex:gemm -c 3 --csv --log-file gpurun_out/r02c/gm${gm}_$pr.csv python tools/kernel_times.py hoc_p8_L1 1 $pr > /dev/null 2>&1
  done
done
echo done
