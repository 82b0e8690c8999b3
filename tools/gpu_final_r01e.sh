# r01e end-of-session pass: GPU tests, smoke, every config's bench line (default steps, CPU
# baseline), the reference arm, launch lists; ncu of the FFNN GEMMs (new capture).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r01e
timeout 900 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/r01e/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r01e/smoke.log 2>&1
for c in bmm2 chain3 ffnn_big attn_big hoc; do
  timeout 600 python bench.py --config $c > gpurun_out/r01e/bench_$c.jsonl 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r01e/launches_$c.csv python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r01e/reference_bmm2.jsonl 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 2 -c 2 -o gpurun_out/r01e/gemm_ffnn python bench.py --config ffnn_big --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/r01e/ncu_gemm_ffnn.log 2>&1
echo done
