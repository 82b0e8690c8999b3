# attention v6 (FA4-order single issuer, K/V ring, named-barrier hand-off): parity + timing
cd $GRAFT_REPO_ROOT
OUT=gpurun_out/r02k
mkdir -p $OUT
timeout 120 python tools/kernel_times.py attn_s_p8_L1 3 bf16 > $OUT/small.txt 2>&1
echo "small rc=$?" >> $OUT/small.txt
timeout 200 python tools/kernel_times.py attn_big_p8_L1 20 bf16 > $OUT/big.txt 2>&1
echo "big rc=$?" >> $OUT/big.txt
timeout 900 python -m pytest tests/test_gpu_fusion_fuzz.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -x -q -p no:cacheprovider -k "attn or attention or fusion or flash or fused" > $OUT/pytest.log 2>&1
echo "pytest rc=$?" >> $OUT/pytest.log
echo done
