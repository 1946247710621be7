python -m pytest tests/test_gpu_ops.py tests/test_gpu_batched.py -m gpu -x -q 2>&1 | tail -3
for cfg in C2 C3 C5; do
python bench.py --config $cfg --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-parity > gpurun_out/plan_$cfg.json 2>/dev/null
done
DR_ATTN_QT=4 python bench.py --config C3 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-parity > gpurun_out/plan_C3_qt4.json 2>/dev/null
DR_ATTN_QT=2 python bench.py --config C3 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-parity > gpurun_out/plan_C3_qt2.json 2>/dev/null
DR_ATTN_QT=1 DR_ATTN_KSPLIT=2 python bench.py --config C2 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-parity > gpurun_out/plan_C2_qt1k2.json 2>/dev/null
for f in gpurun_out/plan_*.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); st={k:round(v['ms_per_step'],4) for k,v in d['stages'].items() if 'attn' in k}
print('$f', d['value'], d['p50_ms'], st)"; done
