# x3 attention v4 (128-key blocks): correctness on small graphs (both CTA modes), timing
cd $GRAFT_REPO_ROOT
make -C oracle -s > /dev/null 2>&1
for args in "256 2 0.125 1" "512 2 4.0 1" "1024 4 1.0 1" "128 1 0.125 1" "256 1 0.0 1"; do
  echo "== $args"
  timeout 60 python tools/x3_attn_debug.py $args | grep "normwise"
  ED_ATTN_X3_CTA=1 timeout 60 python tools/x3_attn_debug.py $args | grep "normwise" | sed 's/^/[1cta]/'
done
for i in 1 2; do
timeout 120 python tools/kernel_times.py attn_big_p8_L1 5 fp32x3
ED_ATTN_X3_CTA=1 timeout 120 python tools/kernel_times.py attn_big_p8_L1 5 fp32x3 | sed 's/^/[1cta] /'
done
