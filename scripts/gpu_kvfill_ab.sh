# A/B of the new slot's K/V placement at C2 (DR_KV_FILL) and the device-path side branch
O=gpurun_out/kvab; mkdir -p $O
for v in "0 1" "1 1" "0 2" "2 1"; do
  set -- $v
  for rep in 1 2; do
  DR_KV_FILL=$1 DR_SLOTKV_SIDE=$2 timeout 300 python bench.py --steps 300 --warmup 10 --no-e2e --no-cpu-baseline > $O/c2_fill$1_side$2_$rep.json 2> $O/c2_fill$1_side$2_$rep.err
  python -c "import json;d=json.loads(open('$O/c2_fill$1_side$2_$rep.json').read().strip().splitlines()[-1]);print('fill',$1,'side',$2,d['value'],d['p50_ms'],d['parity']['pass'],d['gpu_launches'])"
  done
done
DR_KV_FILL=1 timeout 600 python scripts/graph_prefix.py > $O/graph_prefix_fill1.txt 2>&1; cat $O/graph_prefix_fill1.txt
DR_KV_FILL=1 timeout 600 python -m pytest tests -m gpu -q -x -k "slot or memory or c2 or sequence or batched" > $O/pytest_fill1.log 2>&1; tail -3 $O/pytest_fill1.log
