timeout 600 python -m pytest tests/test_gpu_frame_ops.py -x -q 2>&1 | tail -15
timeout 300 python scripts/bench_frame_ops.py > gpurun_out/frame_ops_bench.jsonl 2>&1; cat gpurun_out/frame_ops_bench.jsonl
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv python scripts/bench_frame_ops.py --iters 2 > gpurun_out/frame_ops_ncu.csv 2>&1; tail -5 gpurun_out/frame_ops_ncu.csv
