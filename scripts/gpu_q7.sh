tag=${1:-q7}
./scripts/bin/umma_microbench 2>&1 | grep -E "mode (0|8|9)"
for k in dec_fused_kernel dec_border mask_fused; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 \
    -o gpurun_out/${tag}_$k python scripts/profile_frame.py --config C5 --frames 1 \
    > gpurun_out/${tag}_ncu_$k.log 2>&1; tail -1 gpurun_out/${tag}_ncu_$k.log
done
