# direct (zero-copy) receives for refinement folds: peer tests + overlap tool counts
cd $GRAFT_REPO_ROOT
make -C oracle -s > /dev/null 2>&1

for pl in chain3_p8_L2 chain3_p8_L4 attn_big_p8_L2 ffnn_big_p8_L2; do
  for dr in 1 0; do
    ED_PEER_DIRECT=$dr timeout 300 python tools/peer_overlap.py $pl ${pl##*_L} fp32x3 5 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('$pl direct=$dr', round(d['step_ms'],3), {r:(v['copy_ms'] and round(v['copy_ms'],3), round(v['exposed_ms'],3)) for r,v in d['ranks'].items()})
    else: print(l.rstrip()[:200])
"
  done
done
