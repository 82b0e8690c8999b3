# ncu of the bf16 fused attention kernel (tensor-pipe activity for the round-1 verdict's bar)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r02ap
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_kernel -s 3 -c 1 -o gpurun_out/r02ap/attn_bf16_full python tools/kernel_times.py attn_big_p8_L1 1 bf16 > gpurun_out/r02ap/ncu.log 2>&1
tail -2 gpurun_out/r02ap/ncu.log
