timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
python -c "import json;d=json.load(open('gpurun_out/bench.json'));print(d['value'], {k:v['ms_per_step'] for k,v in d['stages'].items()})"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mask -c 1 -o gpurun_out/mask_full python scripts/profile_frame.py --frames 2 > gpurun_out/ncu_m.log 2>&1
tail -1 gpurun_out/ncu_m.log
