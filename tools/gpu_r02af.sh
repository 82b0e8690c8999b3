cd $GRAFT_REPO_ROOT
for args in "256 2 0.125 1" "512 2 4.0 1" "1024 4 1.0 1" "256 1 0.0 1"; do
  echo "== $args"
  ED_LIB_PATH=paper_2410_02682_b200/build/var/x3nw.so timeout 60 python tools/x3_attn_debug.py $args | grep "normwise"
  ED_ATTN_X3_CTA=1 ED_LIB_PATH=paper_2410_02682_b200/build/var/x3nw.so timeout 60 python tools/x3_attn_debug.py $args | grep "normwise" | sed 's/^/[1cta]/'
done
ED_LIB_PATH=paper_2410_02682_b200/build/var/x3nw.so timeout 120 python tools/kernel_times.py attn_big_p8_L1 5 fp32x3
