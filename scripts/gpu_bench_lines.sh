# Refresh the round-end bench lines (C2 default with e2e + CPU leg, C2 over 1000 frames,
# C3 / C5 / C4), GPU tests, smoke, and the C2 mask-stage capture into gpurun_out/final2/
O=gpurun_out/final2; mkdir -p $O
timeout 600 python bench.py > $O/bench_c2.json 2> $O/bench_c2.err; tail -c 300 $O/bench_c2.json
timeout 600 python bench.py --impl reference > $O/bench_ref_c2.json 2> $O/bench_ref_c2.err; tail -c 200 $O/bench_ref_c2.json
timeout 900 python bench.py --frames 1000 --steps 1000 --warmup 20 --no-e2e --no-cpu-baseline > $O/bench_c2_1000.json 2> $O/bench_c2_1000.err
for c in C3 C5 C4; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 --cpu-seconds 10 > $O/bench_$c.json 2> $O/bench_$c.err
  tail -c 300 $O/bench_$c.json
done
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; tail -2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/ncu_bench_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-parity > $O/ncu_bench.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/traffic.csv python scripts/profile_frame.py --frames 3 > $O/traffic.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mask_fused -s 0 -c 1 -o $O/ncu_C2_mask_fused python scripts/profile_frame.py --config C2 --frames 2 > $O/ncu_C2_mask_fused.log 2>&1
