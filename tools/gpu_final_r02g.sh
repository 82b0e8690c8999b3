# r02g evidence pass: kept DRAM traffic first (so the bench lines report it), GPU suite, smoke,
# the driver's bench lines (ours + reference arm), every config in both modes, launch list,
# ncu --set full of the headline GEMM and of the fp32x3 attention kernel.
cd $GRAFT_REPO_ROOT
OUT=gpurun_out/r02g
mkdir -p $OUT
make -C oracle -s > $OUT/make.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv > $OUT/smi.txt
lscpu > $OUT/lscpu.txt
timeout 1500 python tools/capture_traffic.py $OUT/r02_traffic.json hoc:fp32x3 hoc:bf16 bmm2_repart:fp32x3 bmm2_repart:bf16 bmm2:fp32x3 bmm2:bf16 chain3:fp32x3 chain3:bf16 ffnn_big:fp32x3 ffnn_big:bf16 attn_big:fp32x3 attn_big:bf16 > $OUT/traffic.log 2>&1
cp $OUT/r02_traffic.json profiles/r02_traffic.json
timeout 2700 python -u -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $OUT/bench_reference.jsonl 2> $OUT/bench_reference.err
timeout 900 python bench.py --steps 20 --warmup 5 > $OUT/bench_default.jsonl 2> $OUT/bench_default.err
for c in hoc bmm2 bmm2_repart chain3 ffnn_big attn_big; do
  for pr in fp32x3 bf16; do
    timeout 600 python bench.py --config $c --precision $pr --extras '' --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 6 > $OUT/bench_${c}_$pr.jsonl 2>&1
  done
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_default.csv python bench.py --steps 2 --warmup 1 --extras '' --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_x3 -s 3 -c 1 -o $OUT/hoc_x3_full python tools/kernel_times.py hoc_p8_L1 1 fp32x3 > $OUT/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_x3 -s 3 -c 1 -o $OUT/attn_x3_full python tools/kernel_times.py attn_big_p8_L1 1 fp32x3 > $OUT/ncu_attn_x3.log 2>&1
echo done
