cd $GRAFT_REPO_ROOT
for v in x3p x3e1 x3e2 x3e3 x3e123; do
  echo "== $v"
  ED_LIB_PATH=paper_2410_02682_b200/build/var/$v.so timeout 120 python tools/kernel_times.py attn_big_p8_L1 2 fp32x3 2>&1 | grep "cta 0\|attn_big" | sort | uniq | head -4
done
