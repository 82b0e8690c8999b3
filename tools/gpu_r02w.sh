# fp32x3 fused attention: first run
cd $GRAFT_REPO_ROOT
make -C oracle -s > /dev/null 2>&1
export KT_TOP=8
timeout 120 python tools/kernel_times.py attn_big_p8_L1 5 fp32x3; echo "rc=$?"
ED_ATTN_X3=0 timeout 120 python tools/kernel_times.py attn_big_p8_L1 5 fp32x3 | sed 's/^/[unfused] /'
timeout 600 python -m pytest tests/test_gpu_fullsize.py -x -q -k "attn_big and fp32x3" -s 2>&1 | tail -15
