# End-of-round bench pass: every config with the default step counts and the CPU baseline,
# plus the reference arm on bmm2; launch lists with DRAM bytes; ncu of the headline GEMM.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/prof
for c in bmm2 chain3 ffnn_big attn_big hoc; do
  timeout 600 python bench.py --config $c > gpurun_out/prof/bench_$c.jsonl 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/prof/launches_$c.csv python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/prof/reference_bmm2.jsonl 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 2 -c 2 -o gpurun_out/prof/gemm_bmm2 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/prof/ncu_gemm.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 1 -c 1 -o gpurun_out/prof/gemm_hoc python bench.py --config hoc --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/prof/ncu_gemm_hoc.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_kernel -s 1 -c 1 -o gpurun_out/prof/attn python bench.py --config attn_big --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/prof/ncu_attn.log 2>&1
