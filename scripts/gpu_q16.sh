timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python bench.py --config C5 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/q16_c5.json 2>/dev/null
python -c "import json;d=json.loads(open('gpurun_out/q16_c5.json').read().strip().splitlines()[-1]);print('c5', d['value'], d['p50_ms'], d['parity']['pass'], {k:v['ms_per_step'] for k,v in d['stages'].items()})"
python bench.py --config C3 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/q16_c3.json 2>/dev/null
python -c "import json;d=json.loads(open('gpurun_out/q16_c3.json').read().strip().splitlines()[-1]);print('c3', d['value'], d['p50_ms'], d['parity']['pass'], {k:v['ms_per_step'] for k,v in d['stages'].items()})"
timeout 300 python scripts/token_trace.py --config C5 2>&1 | tail -6
