# full GPU check: pytest -m gpu, then C2 / C5 / C3 bench lines (no e2e / cpu leg).  Tag $1.
tag=${1:-f}
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for c in C2 C5 C3; do
  python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${tag}_$c.json 2>gpurun_out/${tag}_$c.err
  python -c "import json;d=json.loads(open('gpurun_out/${tag}_$c.json').read().strip().splitlines()[-1]);print('$c', d['value'], d['p50_ms'], d['parity']['pass'], {k:v['ms_per_step'] for k,v in d['stages'].items()})" || tail -5 gpurun_out/${tag}_$c.err
done
