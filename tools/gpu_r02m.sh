cd $GRAFT_REPO_ROOT
OUT=gpurun_out/r02m
mkdir -p $OUT
timeout 600 ncu --set full --import-source on --clock-control none -k regex:attn_kernel -c 1 -o $OUT/v6_full python tools/kernel_times.py attn_big_p8_L1 1 bf16 > $OUT/ncu.log 2>&1
echo done
