tag=${1:-q6}
bash scripts/gpu_dec2.sh $tag
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/${tag}_c2.json 2>/dev/null
python -c "import json;d=json.loads(open('gpurun_out/${tag}_c2.json').read().strip().splitlines()[-1]);print('c2', d['value'], d['p50_ms'], d['parity']['pass'], {k:v['ms_per_step'] for k,v in d['stages'].items()})"
