cd $GRAFT_REPO_ROOT
OUT=gpurun_out/r02l
mkdir -p $OUT
timeout 300 python tools/attn_data_probe.py 20 > $OUT/ours.txt 2>&1
timeout 300 python tools/fa4_compare.py 50 > $OUT/fa4_unit.jsonl 2>/dev/null
timeout 300 python tools/fa4_compare.py 50 30 > $OUT/fa4_big.jsonl 2>/dev/null
echo done
