# Round-end measurement set into gpurun_out/final/ (copied to profiles/r02 by hand):
# tests, smoke, the default bench line (C2, e2e, CPU leg), the reference arm, C3/C4/C5,
# C2 over 1000 frames, the driver's ncu launch list, per-stage DRAM traffic, and
# ncu --set full of the top kernels (C5, C2, C4).
set -x
O=gpurun_out/final; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > $O/nvidia_smi.txt
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; tail -2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 600 python bench.py > $O/bench_c2.json 2> $O/bench_c2.err; tail -c 600 $O/bench_c2.json
timeout 600 python bench.py --impl reference > $O/bench_ref_c2.json 2> $O/bench_ref_c2.err; tail -c 300 $O/bench_ref_c2.json
for c in C3 C5 C4; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 --cpu-seconds 10 > $O/bench_$c.json 2> $O/bench_$c.err
  tail -c 300 $O/bench_$c.json
done
timeout 900 python bench.py --frames 1000 --steps 1000 --warmup 20 --no-e2e --no-cpu-baseline > $O/bench_c2_1000.json 2> $O/bench_c2_1000.err
tail -c 300 $O/bench_c2_1000.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/ncu_bench_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-parity > $O/ncu_bench.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/traffic.csv python scripts/profile_frame.py --frames 3 > $O/traffic.log 2>&1
for spec in "C5 attn_tc_kernel 0" "C2 attn_tc_kernel 0" "C5 dec_fused_kernel 0" "C5 token_tc_kernel 1" "C5 mask_fused 0" "C5 dec_border 0" \
            "C4 attn_tc_kernel 0" "C4 token_q_kernel 2" "C2 v2p_tc_kernel 0" "C2 conv3x3_tc_kernel 0" "C2 dec2_gather 0" "C2 token_q_kernel 2" "C2 mask_fused 0"; do
  set -- $spec
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$2 -s $3 -c 1 -o $O/ncu_${1}_$2 python scripts/profile_frame.py --config $1 --frames 2 > $O/ncu_${1}_$2.log 2>&1
  tail -1 $O/ncu_${1}_$2.log
done
