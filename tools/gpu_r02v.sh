# A/B on one box: lo shadow written by producers (default) vs split launch (ED_X3_LO_EPI=0) vs direct-store lo
cd $GRAFT_REPO_ROOT
export KT_TOP=6
for r in 1 2; do
for pl in bmm2_p8_L1 chain3_p8_L1 attn_big_p8_L1 ffnn_big_p8_L1; do
  timeout 300 python tools/kernel_times.py $pl 10 fp32x3
  ED_X3_LO_EPI=0 timeout 300 python tools/kernel_times.py $pl 10 fp32x3 | sed 's/^/[split] /'
  ED_LIB_PATH=paper_2410_02682_b200/build/var/lodirect.so timeout 300 python tools/kernel_times.py $pl 10 fp32x3
done
done
