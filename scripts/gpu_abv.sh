# A/B of experiment builds (VARIANTS="old k2 ..."; "base" = _build): GPU parity tests of each
# non-base build, then C2 bench lines with per-stage attention times
VARIANTS=${VARIANTS:-base}; STEPS=${STEPS:-300}; TESTS=${TESTS:-tests/test_gpu_parity.py}
lib() { if [ $1 = base ]; then echo ""; else echo "DR_B200_LIB=paper_2509_10466_b200/_build_$1/libdrb200.so"; fi; }
for v in $VARIANTS; do
  echo "== parity $v"; env $(lib $v) timeout 600 python -m pytest $TESTS -q -x 2>&1 | tail -2
done
for rep in 1 2; do
for v in $VARIANTS; do
  env $(lib $v) timeout 300 python bench.py --steps $STEPS --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$v', d['value'], d['e2e']['value'] if 'e2e' in d else '', {k:round(v['ms_per_step']*1e3,1) for k,v in d['stages'].items()})"
done
done
