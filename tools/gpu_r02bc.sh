# N > 1 bench path (torchrun, peer transport) as functional checks with ranks sharing the one GPU
cd $GRAFT_REPO_ROOT
OUT=gpurun_out/r02bc
mkdir -p $OUT
make -C oracle -s > /dev/null 2>&1
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29531"
ED_SAME_DEVICE=1 timeout 600 $R --nproc-per-node 2 bench.py --gpus 2 --steps 3 --warmup 3 > $OUT/n2_default.jsonl 2> $OUT/n2_default.err; echo "n2 default rc=$?"
ED_SAME_DEVICE=1 timeout 600 $R --nproc-per-node 2 bench.py --gpus 2 --steps 3 --warmup 3 --config bmm2_repart --precision bf16 --extras '' > $OUT/n2_repart.jsonl 2> $OUT/n2_repart.err; echo "n2 repart rc=$?"
ED_SAME_DEVICE=1 timeout 600 $R --nproc-per-node 4 bench.py --gpus 4 --steps 3 --warmup 3 --config attn_big --precision fp32x3 --extras '' > $OUT/n4_attn.jsonl 2> $OUT/n4_attn.err; echo "n4 attn rc=$?"
timeout 600 $R --nproc-per-node 2 bench.py --impl reference --gpus 2 --steps 3 --warmup 3 > $OUT/n2_reference.jsonl 2> $OUT/n2_reference.err; echo "n2 reference rc=$?"
for f in $OUT/*.jsonl; do echo "== $f"; cut -c1-600 $f; done
tail -3 $OUT/*.err
