# A/B of experiment libraries (_build_<variant>, selected by DR_B200_LIB) against the
# shipped one: C2 (400 steps) and C5 (15 steps), two rounds.  Usage: gpu_ab_lib.sh v1 v2 ...
O=gpurun_out/ablib; mkdir -p $O
for rep in 1 2; do for v in base "$@"; do
  if [ $v = base ]; then unset DR_B200_LIB; else export DR_B200_LIB=$PWD/paper_2509_10466_b200/_build_$v/libdrb200.so; fi
  for c in C2 C5; do
    st=400; [ $c = C5 ] && st=15
    timeout 300 python bench.py --config $c --steps $st --warmup 5 --no-e2e --no-cpu-baseline --no-parity > $O/${c}_$v.json 2> $O/${c}_$v.err
    python -c "import json;d=json.loads(open('$O/${c}_$v.json').read().strip().splitlines()[-1]);print('$v','$c',d['value'],d['p50_ms'])"
  done
done; done
