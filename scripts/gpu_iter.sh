# Iteration check: GPU tests, C2 / C5 bench lines (no e2e / CPU leg), stage times, mask trace
O=gpurun_out/iter; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; tail -3 $O/pytest_gpu.log
for c in C2 C5; do
  st=300; [ $c = C5 ] && st=15
  timeout 600 python bench.py --config $c --steps $st --warmup 5 --no-e2e --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err
  python - <<PY
import json
d=json.loads(open('$O/bench_$c.json').read().strip().splitlines()[-1])
print('$c', d['value'], d['p50_ms'], 'parity', d['parity']['pass'], 'mask', d['stages'].get('mask_stage'))
PY
done
timeout 300 python scripts/mask_trace.py > $O/mask_trace_c2.txt 2>&1; head -12 $O/mask_trace_c2.txt
