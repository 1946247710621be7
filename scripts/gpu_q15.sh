python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --no-parity > gpurun_out/q15_base.json 2>/dev/null
DR_DEC_FUSED=1 python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --no-parity > gpurun_out/q15_fused.json 2>/dev/null
DR_B200_LIB=paper_2509_10466_b200/_build_mth8/libdrb200.so python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --no-parity > gpurun_out/q15_mth8.json 2>/dev/null
for t in base fused mth8; do python -c "import json;d=json.loads(open('gpurun_out/q15_$t.json').read().strip().splitlines()[-1]);print('$t', d['value'], d['p50_ms'], {k:v['ms_per_step'] for k,v in d['stages'].items()})"; done
