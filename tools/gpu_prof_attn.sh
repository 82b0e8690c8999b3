cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_kernel -s 1 -c 1 -o gpurun_out/attn_prof python bench.py --config attn_big --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_attn.log 2>&1
