cd $GRAFT_REPO_ROOT
make -C oracle -s > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -k "attn" -s 2>&1 | grep -o "'O': {[^}]*}" | head -2
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_fusion_fuzz.py -x -q 2>&1 | tail -2
