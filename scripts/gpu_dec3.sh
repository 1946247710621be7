# fused decoder checks: fused vs unfused vs oracle, decoder/batched tests, C5 bench, C2 with
# the fused decoder forced on vs the default, and the C2 / C5 tile traces.  Tag in $1.
tag=${1:-d}
timeout 600 python scripts/dec_check.py > gpurun_out/${tag}_check.txt 2>&1; tail -6 gpurun_out/${tag}_check.txt
timeout 900 python -m pytest tests/test_gpu_batched.py -x -q 2>&1 | tail -2
for v in "C5 0" "C2 0" "C2 1"; do set -- $v
  env $( [ "$2" = 1 ] && echo DR_DEC_FUSED=1 ) python bench.py --config $1 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${tag}_$1_$2.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/${tag}_$1_$2.json').read().strip().splitlines()[-1]);print('$1 fused=$2', d['value'], d['p50_ms'], d['parity']['pass'], {k:v['ms_per_step'] for k,v in d['stages'].items() if k[:3] in ('dec','sea','vec')})"
done
DR_DEC_FUSED=1 timeout 300 python scripts/dec_trace.py --config C2 2>&1 | grep -E "main loop|finish"
timeout 300 python scripts/dec_trace.py --config C5 2>&1 | grep -E "main loop|finish"
