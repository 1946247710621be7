# round measurement: GPU tests, default bench (with CPU baseline), C3/C5 lines, reference
# arm, ncu launch list + traffic, ncu --set full of the dominant kernel
set -x
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/pytest_gpu.log
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/traffic.csv python scripts/profile_frame.py --frames 3 > /dev/null 2>&1
python scripts/ncu_traffic.py gpurun_out/traffic.csv profiles/r01/ncu_traffic.json
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --config C3 --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 600 python bench.py --config C5 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
timeout 600 python bench.py --config C4 --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_tc -s 0 -c 2 -o gpurun_out/attn_full python scripts/profile_frame.py --frames 2 > gpurun_out/ncu_a.log 2>&1
cp profiles/r01/ncu_traffic.json gpurun_out/
cat gpurun_out/pytest_gpu.log
python scripts/graph_prefix.py 2>&1 | tail -13 > gpurun_out/graph_prefix.txt
python scripts/e2e_trace.py > gpurun_out/e2e_trace.txt 2>&1
