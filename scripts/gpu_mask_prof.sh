# ncu --set full (with source) of the fused mask stage at C5 and C2, for the per-line
# instruction / stall breakdown read back here with `ncu -i ... --page source --csv`.
O=gpurun_out/maskprof; mkdir -p $O
for c in C5 C2; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:mask_fused -c 1 \
    -o $O/ncu_${c}_mask python scripts/profile_frame.py --config $c --frames 1 > $O/ncu_${c}_mask.log 2>&1
  tail -2 $O/ncu_${c}_mask.log
done
