# prefetched peer receives: peer tests, then overlap on one GPU (in-process ranks)
cd $GRAFT_REPO_ROOT
OUT=gpurun_out/r02aa
mkdir -p $OUT
rm -f $OUT/overlap.jsonl
make -C oracle -s > /dev/null 2>&1
timeout 1200 python -m pytest tests/test_gpu_peer.py tests/test_gpu_parity.py -x -q > $OUT/peer_tests.txt 2>&1; tail -3 $OUT/peer_tests.txt
for pl in bmm2_repart_p8_L2 bmm2_repart_p8_L4 bmm2_repart_p8_L8 ffnn_big_p8_L2 attn_big_p8_L2; do
  for pf in 1 0; do
    ED_PEER_PREFETCH=$pf timeout 300 python tools/peer_overlap.py $pl ${pl##*_L} bf16 5 >> $OUT/overlap.jsonl 2> $OUT/overlap_${pl}_$pf.err || tail -3 $OUT/overlap_${pl}_$pf.err
  done
done
python - <<'PY'
import json
for l in open('gpurun_out/r02aa/overlap.jsonl'):
    d=json.loads(l)
    rk={r:(round(v['copy_ms'],3),round(v['exposed_ms'],3),v['hidden_frac'] and round(v['hidden_frac'],2)) for r,v in d['ranks'].items()}
    print(d['plan'],'prefetch' if d['prefetch'] else 'at-consumer', round(d['step_ms'],3),'ms', d['peer_bytes_per_step'], rk)
PY
