# why attention's fp32x3 projections (0.52 ms) run slower than chain3's same-size GEMMs (0.44 ms)
cd $GRAFT_REPO_ROOT
OUT=gpurun_out/r02bd
mkdir -p $OUT
M=gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,launch__grid_size,lts__t_bytes.sum
timeout 600 ncu --metrics $M --clock-control none -k regex:gemm_x3 -s 12 -c 4 --csv python tools/kernel_times.py chain3_p8_L1 3 fp32x3 > $OUT/chain3.csv 2>&1
timeout 600 ncu --metrics $M --clock-control none -k regex:gemm_x3 -s 16 -c 4 --csv python tools/kernel_times.py attn_big_p8_L1 3 fp32x3 > $OUT/attn.csv 2>&1
timeout 600 ncu --metrics $M --clock-control base -k regex:gemm_x3 -s 12 -c 4 --csv python tools/kernel_times.py chain3_p8_L1 3 fp32x3 > $OUT/chain3_base.csv 2>&1
timeout 600 ncu --metrics $M --clock-control base -k regex:gemm_x3 -s 16 -c 4 --csv python tools/kernel_times.py attn_big_p8_L1 3 fp32x3 > $OUT/attn_base.csv 2>&1
KT_TOP=8 python tools/kernel_times.py attn_big_p8_L1 10 fp32x3 > $OUT/kt.txt 2>&1
KT_TOP=8 python tools/kernel_times.py chain3_p8_L1 10 fp32x3 >> $OUT/kt.txt 2>&1
cat $OUT/kt.txt
