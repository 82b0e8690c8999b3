# attention A/B sweep (variant builds), attn_big, alternating on one box
cd $GRAFT_REPO_ROOT
OUT=gpurun_out/r02p
mkdir -p $OUT
rm -f $OUT/sweep.txt
for rep in 1 2 3; do
  for v in base d1 d2; do
    if [ $v = base ]; then unset ED_LIB_PATH; else export ED_LIB_PATH=paper_2410_02682_b200/build/var/attn_$v.so; fi
    echo -n "$v " >> $OUT/sweep.txt
    timeout 200 python tools/kernel_times.py attn_big_p8_L1 20 bf16 >> $OUT/sweep.txt 2>&1
  done
done
echo done
