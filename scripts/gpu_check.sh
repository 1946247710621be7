set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
python bench.py --steps 200 --warmup 10 > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -3 gpurun_out/bench.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python scripts/profile_frame.py --frames 3 > gpurun_out/ncu_l.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attention -s 2 -c 1 -o gpurun_out/attn_full python scripts/profile_frame.py --frames 3 > gpurun_out/ncu_f.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mask -c 1 -o gpurun_out/mask_full python scripts/profile_frame.py --frames 2 > gpurun_out/ncu_m.log 2>&1
cat gpurun_out/pytest_gpu.log; cat gpurun_out/bench.json
