set -x
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
cat gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
cat gpurun_out/bench.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_tc.csv python scripts/profile_frame.py --frames 3 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:token_tc -s 4 -c 1 -o gpurun_out/tok_full python scripts/profile_frame.py --frames 3 > gpurun_out/ncu_t.log 2>&1
tail -3 gpurun_out/ncu_t.log
