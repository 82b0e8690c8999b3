# A/B: GEMM MMA issue from one lane (old) vs warp-wide elected (new), same box, alternating
cd $GRAFT_REPO_ROOT
OUT=gpurun_out/r02o
mkdir -p $OUT
for rep in 1 2 3; do
  for v in new old; do
    if [ $v = old ]; then export ED_LIB_PATH=paper_2410_02682_b200/build/var/gemm_lane.so; else unset ED_LIB_PATH; fi
    for c in bmm2 chain3 ffnn_big hoc; do
      echo -n "$v " >> $OUT/ab.txt
      timeout 300 python tools/kernel_times.py ${c}_p8_L1 10 bf16 >> $OUT/ab.txt 2>&1
    done
    echo -n "$v " >> $OUT/ab.txt
    timeout 300 python tools/kernel_times.py chain3_p8_L1 10 fp32x3 >> $OUT/ab.txt 2>&1
  done
done
echo done
