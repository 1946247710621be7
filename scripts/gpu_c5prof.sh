# C5 captures: ncu --set full of the mask stage and the fused decoder kernels (one launch
# each, batch 64), then the PyTorch-eager yardstick.  Tag in $1.
tag=${1:-c5}
python scripts/profile_frame.py --config C5 --frames 1 > gpurun_out/${tag}_plain.log 2>&1 || { cat gpurun_out/${tag}_plain.log; exit 1; }
for k in mask_fused dec_fused_kernel dec_border dec_fixup; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 \
    -o gpurun_out/${tag}_$k python scripts/profile_frame.py --config C5 --frames 1 \
    > gpurun_out/${tag}_ncu_$k.log 2>&1; tail -1 gpurun_out/${tag}_ncu_$k.log
done
timeout 900 python scripts/eager_yardstick.py --steps 20 > gpurun_out/${tag}_eager.json 2> gpurun_out/${tag}_eager.err
cat gpurun_out/${tag}_eager.json; tail -3 gpurun_out/${tag}_eager.err
