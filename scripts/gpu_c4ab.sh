for v in 0 1; do
  env $( [ "$v" = 1 ] && echo DR_DEC_FUSED=1 ) python bench.py --config C4 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c4ab_$v.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/c4ab_$v.json').read().strip().splitlines()[-1]);print('fused=$v', d['value'], d['p50_ms'], d['parity']['pass'], {k:v['ms_per_step'] for k,v in d['stages'].items()})"
done
