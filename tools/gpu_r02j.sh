# attention calibration: public Blackwell attention kernels vs the fused kernel on attn_big's shape
cd $GRAFT_REPO_ROOT
OUT=gpurun_out/r02j
mkdir -p $OUT
timeout 600 python tools/fa4_compare.py 50 > $OUT/fa4.jsonl 2> $OUT/fa4.err
timeout 300 python tools/kernel_times.py attn_big_p8_L1 20 bf16 > $OUT/ours.txt 2>&1
timeout 600 ncu --set full --clock-control none -k regex:flash_fwd -c 1 -o $OUT/fa4_full python tools/fa4_compare.py 3 > $OUT/ncu_fa4.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:attn_kernel -c 1 -o $OUT/ours_full python tools/kernel_times.py attn_big_p8_L1 1 bf16 > $OUT/ncu_ours.log 2>&1
echo done
