cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python tools/debug_vertices.py ffnn_big_p8_L1 > gpurun_out/dbg_ffnn.log 2>&1
timeout 600 python tools/debug_vertices.py attn_big_p8_L1 > gpurun_out/dbg_attn.log 2>&1
