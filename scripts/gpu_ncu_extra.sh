O=gpurun_out/extra; mkdir -p $O
for spec in "C4 attn_tc_kernel 0" "C4 token_q_kernel 2" "C2 v2p_tc_kernel 0" "C2 conv3x3_tc_kernel 0" "C2 dec2_gather 0" "C2 token_q_kernel 2" "C2 mask_fused 0"; do
  set -- $spec
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$2 -s $3 -c 1 -o $O/ncu_${1}_$2 python scripts/profile_frame.py --config $1 --frames 2 > $O/ncu_${1}_$2.log 2>&1
  tail -1 $O/ncu_${1}_$2.log
done
