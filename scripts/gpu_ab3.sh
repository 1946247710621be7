# parity of two experiment builds + C2 bench of base and both
for v in ex2h ex2h8; do
  echo "== $v"; DR_B200_LIB=paper_2509_10466_b200/_build_$v/libdrb200.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
done
for v in base ex2h ex2h8; do
  if [ $v = base ]; then L=""; else L="DR_B200_LIB=paper_2509_10466_b200/_build_$v/libdrb200.so"; fi
  env $L timeout 300 python bench.py --steps 300 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$v', d['value'], {k:round(v['ms_per_step']*1e3,1) for k,v in d['stages'].items() if 'attn' in k})"
done
