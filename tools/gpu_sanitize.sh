# compute-sanitizer over one small case per kernel class (tcgen05 GEMM in
# bf16 / tf32 / fp32x3 with lo shadows and split tiles, fused attention bf16 and
# fp32x3, softmax rows, refine/rect folds, generic fp64, peer transport):
# memcheck, racecheck (shared memory), synccheck (barriers), initcheck.
# Logs under gpurun_out/sanitize/; the summary lines go to profiles/.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/sanitize
CASES="attn_s_p8_L1:fp32x3 attn_s_p8_L1:bf16 ffnn_s_p8_L1:fp32x3 ffnn_s_p8_L1:bf16 hoc_s_p8_L1:fp32x3 chain3_s_p8_L1:tf32 bmm2_s_repart_p8_L1:fp32x3 attention_p8_L4:fp64 mix_p4_L2:fp32"
for tool in memcheck racecheck synccheck initcheck; do
  for c in $CASES; do
    name=${c%%:*}; prec=${c##*:}
    log=gpurun_out/sanitize/${tool}_${name}_${prec}.log
    timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/gpu_case.py $name $prec > $log 2>&1
    echo "$tool $name $prec rc=$? | $(grep -h 'CASE ' $log | tail -1) | $(grep -h 'SUMMARY' $log | tr '\n' ' ')" | tee -a gpurun_out/sanitize/summary.txt
  done
done
