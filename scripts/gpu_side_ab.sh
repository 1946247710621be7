# A/B of the slot K/V side branch (DR_SLOTKV_SIDE): tests, then C2 device + e2e, interleaved.
tag=${1:-side}
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for rep in 1 2; do
  for sd in 0 1; do
    DR_SLOTKV_SIDE=$sd timeout 600 python bench.py --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/${tag}_${sd}_$rep.json 2>gpurun_out/${tag}_${sd}_$rep.err
    python -c "import json;d=json.loads(open('gpurun_out/${tag}_${sd}_$rep.json').read().strip().splitlines()[-1]);e=d.get('e2e') or {};print('side=$sd', d['value'], d['p50_ms'], d['parity']['pass'], e.get('value'), (e.get('dropin') or {}).get('value') if isinstance(e.get('dropin'),dict) else e.get('dropin_value'))" || tail -5 gpurun_out/${tag}_${sd}_$rep.err
  done
done
