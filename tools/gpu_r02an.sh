# bf16 attention in cta_group::2 pairs: A/B timing, attention tests
cd $GRAFT_REPO_ROOT
make -C oracle -s > /dev/null 2>&1
for i in 1 2; do
timeout 120 python tools/kernel_times.py attn_big_p8_L1 20 bf16
ED_ATTN_CTA=1 timeout 120 python tools/kernel_times.py attn_big_p8_L1 20 bf16 | sed 's/^/[1cta] /'
done
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_fusion_fuzz.py tests/test_gpu_parity.py -x -q -k "attn or attention or fusion" 2>&1 | tail -2
