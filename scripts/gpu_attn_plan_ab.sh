# C2: forced attention plans (DR_ATTN_QT x DR_ATTN_KSPLIT, every launch) vs the planner
O=gpurun_out/plan; mkdir -p $O
for v in "0 0" "4 4" "2 4" "4 2" "2 2" "1 2" "0 0"; do
  set -- $v
  DR_ATTN_QT=$1 DR_ATTN_KSPLIT=$2 timeout 300 python bench.py --steps 400 --warmup 10 --no-e2e --no-cpu-baseline --no-parity > $O/c2_$1_$2.json 2> $O/c2_$1_$2.err
  python -c "import json;d=json.loads(open('$O/c2_$1_$2.json').read().strip().splitlines()[-1]);s=d['stages'];print('qt',$1,'k',$2,d['value'],d['p50_ms'],s['attn_spatial']['ms_per_step'],s['attn_temporal']['ms_per_step'])"
done
