# fused fp32x3 attention: targeted tests, then the whole GPU suite
cd $GRAFT_REPO_ROOT
OUT=gpurun_out/r02z
mkdir -p $OUT
make -C oracle -s > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -k "attn" -s > $OUT/fullsize_attn.txt 2>&1; echo "rc=$?" >> $OUT/fullsize_attn.txt
grep -E "attn_big|passed|failed|Error" $OUT/fullsize_attn.txt | cut -c1-600
timeout 900 python -m pytest tests/test_gpu_fusion_fuzz.py -x -q > $OUT/fuzz.txt 2>&1; tail -3 $OUT/fuzz.txt
timeout 1800 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.txt 2>&1; tail -3 $OUT/pytest_gpu.txt
