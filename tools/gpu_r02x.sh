cd $GRAFT_REPO_ROOT
make -C oracle -s > /dev/null 2>&1
for args in "256 2 0.125 1" "128 1 0.125 1" "256 1 0.0 1" "512 2 0.125 1" "512 2 4.0 1" "1024 4 1.0 1" "512 2 0.125 2"; do
  echo "== $args"
  timeout 120 python tools/x3_attn_debug.py $args | grep "normwise"
done
timeout 120 python tools/kernel_times.py attn_big_p8_L1 5 fp32x3
ED_LIB_PATH=paper_2410_02682_b200/build/var/x3p.so timeout 120 python tools/kernel_times.py attn_big_p8_L1 1 fp32x3 2>&1 | grep "cta 0"
