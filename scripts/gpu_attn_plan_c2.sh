# C2 attention plan sweep (DR_ATTN_QT / DR_ATTN_KSPLIT overrides) vs the cost-model choice
for v in "0 0" "4 2" "2 4" "2 2" "1 2" "4 4"; do set -- $v
  env $( [ "$1" != 0 ] && echo DR_ATTN_QT=$1 DR_ATTN_KSPLIT=$2 ) python bench.py --steps 100 --warmup 10 --no-cpu-baseline --no-e2e --no-parity > gpurun_out/plan2_$1_$2.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/plan2_$1_$2.json').read().strip().splitlines()[-1]);print('qt=$1 k=$2', d['value'], d['p50_ms'], {k:v['ms_per_step'] for k,v in d['stages'].items() if 'attn' in k})"
done
