# x3 region fusion up to kMaxSib siblings: kernel lists, parity
cd $GRAFT_REPO_ROOT
make -C oracle -s > /dev/null 2>&1
export KT_TOP=8
for pl in attn_big_p8_L1 ffnn_big_p8_L1 chain3_p8_L1 bmm2_repart_p8_L1 hoc_p8_L1; do timeout 300 python tools/kernel_times.py $pl 5 fp32x3; done
timeout 1200 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_fusion_fuzz.py -x -q 2>&1 | tail -2
