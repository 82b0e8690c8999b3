# r02a: TF32 peak, fp32x3 / bf16 bench lines for hoc and bmm2_repart (state at round start)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r02a
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/r02a/smi.txt
lscpu > gpurun_out/r02a/lscpu.txt
timeout 300 python tools/measure_peaks_tf32.py gpurun_out/r02a/tf32_peak.json > gpurun_out/r02a/tf32.log 2>&1
for c in hoc bmm2_repart bmm2 chain3; do
  for p in fp32x3 bf16; do
    timeout 600 python bench.py --config $c --precision $p --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/r02a/bench_${c}_$p.jsonl 2>&1
  done
done
echo done
