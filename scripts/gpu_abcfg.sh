# C3 / C5 bench lines of each build in VARIANTS ("base" = _build), attention stages only
VARIANTS=${VARIANTS:-base}
lib() { if [ $1 = base ]; then echo ""; else echo "DR_B200_LIB=paper_2509_10466_b200/_build_$1/libdrb200.so"; fi; }
for cfg in ${CFGS:-C3 C5}; do
for v in $VARIANTS; do
  if [ $cfg = C5 ]; then S="--steps 8 --warmup 3"; else S="--steps 50 --warmup 5"; fi
  env $(lib $v) timeout 600 python bench.py --config $cfg $S --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$cfg $v', d['value'], {k:round(v['ms_per_step']*1e3,1) for k,v in d['stages'].items() if 'attn' in k})"
done
done
